// internal.h -- host-side declarations shared by the .cu translation units of
// librbe_cuda.so (not part of the public C ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "rbe_common.cuh"

namespace rbe_dev {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define RBE_CK(expr)                                                                          \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            throw ::rbe_dev::CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                       " at " __FILE__ ":" + std::to_string(__LINE__));       \
    } while (0)

// Index-wide constants every kernel needs.
struct Shape {
    uint32_t dim = 0;
    uint32_t kp = 1;
    uint32_t rw = 1;
    uint32_t wpp = 1;  // u64 words per plane (reference)
    uint32_t w32 = 2;  // u32 words per plane (device)
};

// Per-plane bit permutation of the device layout: device bit P of word g of
// plane t holds natural dim 32*g + perm[t][P].
struct PlanePerm {
    uint8_t perm[kMaxPlanes][32];
};
PlanePerm derive_plane_permutation(uint32_t kp, bool rw);

// ---- index kernels (index_kernels.cu)
void launch_repack_planes(const uint64_t* d_natural, uint32_t* d_dev, uint64_t count, uint64_t count_pad,
                          const Shape& s, const PlanePerm& perm, cudaStream_t st);
void launch_unpack_planes(const uint32_t* d_dev, uint64_t* d_natural, uint64_t count, uint64_t count_pad,
                          const Shape& s, const PlanePerm& perm, cudaStream_t st);
void launch_fill_synthetic(uint32_t* d_planes, float* d_mags, uint64_t* d_ids, uint64_t count,
                           uint64_t count_pad, uint32_t ordinal, uint32_t n_parts_total, uint64_t n_total,
                           uint64_t seed, const Shape& s, const PlanePerm& perm, cudaStream_t st);
void launch_validate_mags(const float* d_mags, uint64_t count, uint32_t* d_bad, cudaStream_t st);
// d_out[0] += number of i with sorted[i] == sorted[i + 1]
void launch_count_adjacent_equal(const uint64_t* d_sorted, uint64_t n, uint32_t* d_out, cudaStream_t st);
// RBEE records (raw, 4-byte aligned) -> the partitions of a handle (IndexBuilder::add semantics);
// d_bad[0]: magnitudes still not > 0 after the recompute, d_bad[1]: non-finite magnitudes
void launch_rbee_scatter(const uint32_t* d_records, uint64_t rec0, uint64_t n, uint32_t P, const int32_t* d_local,
                         const PartDesc* d_parts, const Shape& s, const PlanePerm& perm, uint32_t* d_bad,
                         cudaStream_t st);
void launch_fill_f32(float* p, uint64_t n, float v, cudaStream_t st);
// d_out[0] = min, d_out[1] = max magnitude bits (caller initialises to ~0u / 0)
void launch_mag_range(const float* d_mags, uint64_t count, uint32_t* d_out, cudaStream_t st);

// ---- per-batch query preparation (scan_exact.cu)
// natural query words [Q][qp][wpp] u64 -> permuted u32 words for the exact
// kernel: [Q][kp][qp][W32] (plane s permuted with doc plane t's permutation).
void launch_prepare_queries_exact(const uint64_t* d_q, uint32_t* d_qperm, uint32_t Q, uint32_t qp,
                                  const Shape& s, const PlanePerm& perm, cudaStream_t st);

struct ScanArgs {
    const PartDesc* parts = nullptr;  // device array
    uint32_t n_parts = 0;
    uint32_t blocks = 1, tpb = 256, ipt = 256, ql = 1;
    uint32_t Q = 0, qp = 1;
    uint64_t max_threads = 0;      // max over partitions of logical threads actually used
    Result* surv = nullptr;        // [Q][surv_cap]
    unsigned long long* surv_count = nullptr;  // [Q]
    uint64_t surv_cap = 0;
    unsigned long long* scored = nullptr;      // [1]
    unsigned int* overflow = nullptr;          // [1]
    unsigned int* error = nullptr;             // [1] internal consistency failures (tensor scan)
    float mag_lo = 0.0f, mag_hi = 0.0f;        // magnitude range of the index (tensor threshold bins)
    // local_select output (exact kernel, one query, one partition): per logical thread
    // t = block * T_b + thread its list [t * ql_eff, + list_counts[t]) of (score, slot),
    // ordered by (score desc, slot asc) like BoundedQueue (search.cpp:32-48)
    double* list_scores = nullptr;
    uint64_t* list_slots = nullptr;
    uint32_t* list_counts = nullptr;
};

// ---- exact kernel (scan_exact.cu)
void launch_scan_exact(const ScanArgs& a, const Shape& s, const uint32_t* d_qperm, void* d_queue_scratch,
                       cudaStream_t st);
size_t exact_queue_scratch_bytes(const ScanArgs& a);

// ---- selection (select.cu): top-n per query of the survivor lists under
// (score desc, id asc).  in: [Q][cap] with counts[Q]; out: [Q][n].
void launch_select_topn(const Result* d_in, const unsigned long long* d_counts, uint64_t cap, uint32_t Q,
                        uint64_t n, Result* d_out, void* d_scratch, size_t scratch_bytes, cudaStream_t st);
size_t select_scratch_bytes(uint32_t Q, uint64_t cap, uint64_t n);
// Result records -> caller SoA arrays (device or pinned host memory), counts per query.
void launch_results_to_soa(const Result* d_in, uint32_t Q, uint64_t n, double* S, uint64_t* I, uint32_t* P,
                           int64_t* A, uint64_t* C, cudaStream_t st);

}  // namespace rbe_dev
