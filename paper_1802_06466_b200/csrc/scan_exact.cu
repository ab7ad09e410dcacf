// scan_exact.cu -- the EXACT scan variant: a literal CUDA-core restatement of
// local_select (src/search.cpp:57-113).  One CUDA thread per (logical thread
// (x, y) of Algorithm 1, group of 4 queries); XOR + __popc per plane pair
// (binary_dot_words, binary_vector.hpp:33-40), the scaled integer
// accumulator of combine_plane_dots (src/embedding.cpp:38-58), the IEEE
// double score ldexp(acc, -L) / double(mag) (__ddiv_rn == x86 divsd), and
// the BoundedQueue of search.cpp:32-48 (strict > to displace, equal scores
// after existing ones).  It is the general kernel (any geometry, queue
// length, plane count, dim) and the full-scale GPU cross-check of the
// TENSOR variant.
#include <cuda_runtime.h>

#include "internal.h"

namespace rbe_dev {
namespace {

constexpr int kQG = 4;          // queries per CUDA thread
constexpr int kThreads = 128;   // CUDA threads per CTA

struct QueueEntry {
    double score;
    uint64_t slot;
    int64_t acc;
};

// natural [Q][qp][wpp] u64 -> [Q][kp][qp][W32] u32, query plane s permuted with
// doc plane t's permutation so popc(q ^ k) is taken over matching dims.
__global__ void prepare_queries_exact_kernel(const uint64_t* __restrict__ q, uint32_t* __restrict__ out, uint32_t Q,
                                             uint32_t qp, uint32_t kp, uint32_t wpp, PlanePerm perm) {
    const uint32_t w32 = 2 * wpp;
    const uint64_t total = uint64_t(Q) * kp * qp * w32;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t g = uint32_t(e % w32);
        const uint32_t s = uint32_t((e / w32) % qp);
        const uint32_t t = uint32_t((e / (uint64_t(w32) * qp)) % kp);
        const uint32_t qi = uint32_t(e / (uint64_t(w32) * qp * kp));
        const uint64_t v = q[(uint64_t(qi) * qp + s) * wpp + (g >> 1)];
        const uint32_t nat = (g & 1) ? uint32_t(v >> 32) : uint32_t(v);
        uint32_t d = 0;
        for (int b = 0; b < 32; ++b) d |= ((nat >> perm.perm[t][b]) & 1u) << b;
        out[e] = d;
    }
}

__device__ __forceinline__ void queue_insert(QueueEntry* q, uint32_t& size, uint32_t cap, double score, uint64_t slot,
                                             int64_t acc) {
    if (size == cap) {
        if (score <= q[size - 1].score) return;  // equal keeps the earlier slot
        --size;
    }
    // upper_bound: first entry with score > entry.score, shifting the tail.
    uint32_t pos = 0;
    while (pos < size && !(score > q[pos].score)) ++pos;
    for (uint32_t k = size; k > pos; --k) q[k] = q[k - 1];
    q[pos] = QueueEntry{score, slot, acc};
    ++size;
}

template <int QG>
__global__ void __launch_bounds__(kThreads) scan_exact_kernel(ScanArgs a, uint32_t dim, uint32_t kp, uint32_t rw,
                                                              uint32_t w32, const uint32_t* __restrict__ qperm,
                                                              QueueEntry* __restrict__ scratch, uint32_t ql_eff) {
    extern __shared__ uint32_t sq[];  // [QG][kp][qp][w32]
    const uint32_t qp = a.qp;
    const uint32_t q0 = blockIdx.z * QG;
    const uint32_t per_q = kp * qp * w32;
    for (uint32_t e = threadIdx.x; e < QG * per_q; e += blockDim.x) {
        const uint32_t qi = q0 + e / per_q;
        sq[e] = qi < a.Q ? qperm[uint64_t(qi) * per_q + e % per_q] : 0u;
    }
    __syncthreads();

    const PartDesc part = a.parts[blockIdx.y];
    const uint64_t n_threads = uint64_t(a.blocks) * a.tpb;
    const uint64_t gt = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint64_t scored = 0;
    if (gt < n_threads) {
        const uint64_t x = gt / a.tpb, y = gt % a.tpb;
        const int L = rw ? int(qp + kp - 2) : 0;
        QueueEntry best[QG];
        uint32_t size[QG];
        QueueEntry* qs[QG];
#pragma unroll
        for (int j = 0; j < QG; ++j) {
            size[j] = 0;
            best[j] = QueueEntry{0.0, 0, 0};
            qs[j] = scratch ? scratch + ((uint64_t(q0 + j) * a.n_parts + blockIdx.y) * n_threads + gt) * ql_eff
                            : nullptr;
        }
        uint64_t z = x * a.tpb * a.ipt + y;
        for (uint32_t i = 0; i < a.ipt; ++i, z += a.tpb) {
            if (z >= part.count) break;  // z grows with i: the rest is out of range too
            int64_t acc[QG];
#pragma unroll
            for (int j = 0; j < QG; ++j) acc[j] = 0;
            const bool il = interleaved_store(int(kp), rw != 0);
            for (uint32_t t = 0; t < kp; ++t) {
                const uint32_t* dw = part.planes + (uint64_t(t) * part.count_pad + z) * w32;
                for (uint32_t s = 0; s < qp; ++s) {
                    int mism[QG];
#pragma unroll
                    for (int j = 0; j < QG; ++j) mism[j] = 0;
                    for (uint32_t g = 0; g < w32; ++g) {
                        uint32_t d;
                        if (il) {  // plane-interleaved store: recover plane t's word of group g
                            uint32_t zz[3], pw[3];
                            for (uint32_t c = 0; c < 3; ++c)
                                zz[c] = __ldg(part.planes + (uint64_t(c) * part.count_pad + z) * w32 + g);
                            deinterleave3(zz, pw);
                            d = pw[t];
                        } else {
                            d = __ldg(dw + g);
                        }
#pragma unroll
                        for (int j = 0; j < QG; ++j) mism[j] += __popc(sq[((j * kp + t) * qp + s) * w32 + g] ^ d);
                    }
                    // dots[s][t] = dim - 2 * mismatches; Horner over levels l = s + t
                    // equals sum dots[s][t] * 2^(L - s - t) exactly in integers.
                    const int sh = rw ? L - int(s + t) : 0;
#pragma unroll
                    for (int j = 0; j < QG; ++j) acc[j] += (int64_t(dim) - 2 * int64_t(mism[j])) << sh;
                }
            }
            const double mag = double(__ldg(part.mags + z));
#pragma unroll
            for (int j = 0; j < QG; ++j) {
                if (q0 + j >= a.Q) continue;
                const double score = __ddiv_rn(ldexp(double(acc[j]), -L), mag);
                if (ql_eff == 1) {
                    if (size[j] == 0 || score > best[j].score) {
                        best[j] = QueueEntry{score, z, acc[j]};
                        size[j] = 1;
                    }
                } else {
                    queue_insert(qs[j], size[j], ql_eff, score, z, acc[j]);
                }
            }
            ++scored;
        }
        if (a.list_counts) {  // local_select: the per-thread lists themselves (query 0)
            a.list_counts[gt] = size[0];
            for (uint32_t k = 0; k < size[0]; ++k) {
                const QueueEntry& e = ql_eff == 1 ? best[0] : qs[0][k];
                a.list_scores[gt * ql_eff + k] = e.score;
                a.list_slots[gt * ql_eff + k] = e.slot;
            }
        }
#pragma unroll
        for (int j = 0; j < QG; ++j) {
            const uint32_t qi = q0 + j;
            if (qi >= a.Q || a.list_counts) continue;
            for (uint32_t k = 0; k < size[j]; ++k) {
                const QueueEntry& e = ql_eff == 1 ? best[j] : qs[j][k];
                const unsigned long long pos = atomicAdd(a.surv_count + qi, 1ull);
                if (pos < a.surv_cap) {
                    Result r;
                    r.score = e.score;
                    r.id = part.ids[e.slot];
                    r.acc = e.acc;
                    r.partition = part.ordinal;
                    r.valid = 1;
                    a.surv[uint64_t(qi) * a.surv_cap + pos] = r;
                } else {
                    atomicExch(a.overflow, 1u);
                }
            }
        }
    }
    // exhaustiveness counter (SearchStats::scored): items scored x queries of the group
    scored *= uint64_t(min(uint32_t(QG), a.Q - q0));
    for (int off = 16; off > 0; off >>= 1) scored += __shfl_down_sync(0xffffffffu, scored, off);
    if ((threadIdx.x & 31) == 0 && scored) atomicAdd(a.scored, (unsigned long long)scored);
}

}  // namespace

void launch_prepare_queries_exact(const uint64_t* d_q, uint32_t* d_qperm, uint32_t Q, uint32_t qp, const Shape& s,
                                  const PlanePerm& perm, cudaStream_t st) {
    const uint64_t total = uint64_t(Q) * s.kp * qp * s.w32;
    if (!total) return;
    uint64_t g = (total + 255) / 256;
    prepare_queries_exact_kernel<<<unsigned(g < 65535 ? g : 65535), 256, 0, st>>>(d_q, d_qperm, Q, qp, s.kp, s.wpp,
                                                                                 perm);
    RBE_CK(cudaGetLastError());
}

size_t exact_queue_scratch_bytes(const ScanArgs& a) {
    const uint64_t ql_eff = a.ql < a.ipt ? a.ql : a.ipt;
    if (ql_eff <= 1) return 0;
    const uint64_t qpad = (uint64_t(a.Q) + kQG - 1) / kQG * kQG;
    return size_t(qpad * a.n_parts * uint64_t(a.blocks) * a.tpb * ql_eff * sizeof(QueueEntry));
}

void launch_scan_exact(const ScanArgs& a, const Shape& s, const uint32_t* d_qperm, void* d_queue_scratch,
                       cudaStream_t st) {
    const uint32_t ql_eff = a.ql < a.ipt ? a.ql : a.ipt;
    const uint64_t n_threads = uint64_t(a.blocks) * a.tpb;
    const uint64_t gx = (n_threads + kThreads - 1) / kThreads;
    if (gx > 0x7fffffffull) throw std::invalid_argument("search: geometry too large for the exact kernel");
    const size_t smem = size_t(kQG) * s.kp * a.qp * s.w32 * sizeof(uint32_t);
    if (smem > 200 * 1024) throw std::invalid_argument("search: query too large for the exact kernel");
    auto kern = scan_exact_kernel<kQG>;
    RBE_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    dim3 grid(unsigned(gx), a.n_parts, (a.Q + kQG - 1) / kQG);
    kern<<<grid, kThreads, smem, st>>>(a, s.dim, s.kp, s.rw, s.w32, d_qperm,
                                       static_cast<QueueEntry*>(d_queue_scratch), ql_eff);
    RBE_CK(cudaGetLastError());
}

}  // namespace rbe_dev
