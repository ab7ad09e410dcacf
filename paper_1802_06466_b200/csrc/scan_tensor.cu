// scan_tensor.cu -- the TENSOR scan variant: tcgen05 int8 tensor-core scoring
// of every (query, doc) pair with the rbeKNN per-logical-thread selection
// fused behind a conservative per-query threshold.
//
// Algebra.  For a query with qp planes and a doc with kp planes, the
// reference's scaled integer accumulator (combine_plane_dots,
// src/embedding.cpp:38-58 over binary_dot_words, binary_vector.hpp:33-40)
// equals, summing over ALL 64*wpp bit positions j (pad bits included, as the
// reference never masks them):
//   weighted:   acc = sum_j (2 rq_j) V_j - (2^kp - 1) sum_j rq_j - pad (2^qp-1)(2^kp-1)
//               rq_j = sum_s 2^(qp-1-s)(2q_s[j]-1),  V_j = sum_t 2^(kp-1-t) k_t[j]
//   unweighted: acc = sum_j (2 ru_j) U_j - kp sum_j ru_j - pad qp kp
//               ru_j = sum_s (2q_s[j]-1),            U_j = sum_t k_t[j]
// so acc = D + C_q with D = (s8 query bytes) x (u8 doc bytes) on the tensor
// cores (tcgen05.mma kind::i8, s32 accumulators in TMEM) and C_q a per-query
// constant.  The doc bytes V_j are produced from the bit-plane-major store by
// the expand32 bit tricks (rbe_common.cuh) straight into TMEM (tcgen05.st),
// which is the MMA's A operand.
//
// Selection.  Algorithm 1 keeps, per logical thread (x, y), its best
// queue_length(=1) items (search.cpp:32-48, 57-113); only the top n survivors
// per query matter (search.cpp:115-128, 160-167).  A probe pass over the first
// `probe_tiles` tiles of every logical block gives, per query, the n-th largest
// of per-thread maxima over distinct threads -- a lower bound theta_q on the
// final n-th survivor score.  Items scoring below theta_q can neither be in
// the top n nor change which items >= theta_q survive, so the main pass keeps
// a per-(query, thread) queue only for the pairs that pass an integer
// threshold test on D (one ISETP per pair); those few are scored exactly in
// FP64 (IEEE division, bit-identical to the CPU) and ranked with the
// reference's tie rules.  Scores of all other pairs never leave the SM.
//
// Kernel anatomy (one CTA per SM, persistent over 128-doc "strips" = the
// 128 logical threads y in [128h, 128h+128) of logical block x):
//   warp 8        producer: cp.async.bulk of each sub-tile's plane words into
//                 a shared-memory ring (mbarrier complete_tx); TMEM allocator
//   warp 9        MMA issuer: tcgen05.mma.cta_group::1.kind::i8, A (docs) from
//                 TMEM, B (queries) from shared memory, D double-buffered
//   warps 0-3     expanders: bit planes -> u8 V bytes -> tcgen05.st into A
//   warps 4-7     epilogue: tcgen05.ld of D, threshold filter, exact FP64
//                 rescoring + per-thread queue in shared memory, survivor
//                 emission at strip end
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "scan_tensor.h"

namespace rbe_dev {
namespace {

constexpr int kStages = 6;
constexpr int kThreads = 320;
constexpr int kEpiBar = 1;           // named barrier id for the 128 epilogue threads
constexpr int kQPass = 64;           // queries per pass (state is [64][128] in shared memory)
constexpr uint32_t kEmpty = 0xffffffffu;
constexpr int kProbeTop = 4;         // per-(query, strip) values kept by the probe

struct TensorParams {
    const PartDesc* parts;
    const uint64_t* strip_prefix;  // [n_parts + 1] cumulative strip counts
    uint32_t n_parts;
    uint32_t tpb, ipt;
    uint32_t w32;                  // u32 words per doc plane
    uint32_t q0, nq;               // query range of this pass
    uint32_t n_pad;                // MMA N (multiple of 16, >= nq)
    uint32_t L;                    // 2^-L scale (qp + kp - 2, or 0 unweighted)
    const uint8_t* bimg;           // [nq_total][...] pre-laid-out B image for this pass
    const int32_t* cq;             // [Q] query constants
    const double* theta;           // [Q] exact-score threshold (main pass)
    const double* t2l;             // [Q] theta * 2^L (main pass)
    uint32_t probe_tiles;          // probe pass: tiles per strip (0 = main pass)
    float* probe_out;              // [Q][n_strips * kProbeTop]
    uint64_t n_strips;
    Result* surv;
    unsigned long long* surv_count;
    uint64_t surv_cap;
    unsigned long long* scored;
    unsigned long long* candidates;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// K-major, SWIZZLE_NONE smem matrix descriptor (canonical ((8,n),2):((1,SBO),LBO)
// in 16-byte units): core matrices of 8 rows x 16 B; LBO = 128 B between the
// two 16-byte K chunks of a 32-byte K block, SBO = 256 B between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3fffu);
    d |= uint64_t(128 >> 4) << 16;  // leading byte offset
    d |= uint64_t(256 >> 4) << 32;  // stride byte offset
    d |= uint64_t(1) << 46;         // descriptor version (Blackwell)
    return d;                       // base offset 0, layout SWIZZLE_NONE
}

// instruction descriptor: D s32, A u8 (doc V bytes), B s8 (query 2*rq), K-major both
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N) {
    return (2u << 4) | (0u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

struct StripInfo {
    uint32_t part;
    uint64_t x, h;
    uint32_t n_tiles;
};

__device__ __forceinline__ StripInfo strip_info(const TensorParams& p, uint64_t s) {
    StripInfo si{0, 0, 0, 0};
    uint32_t part = 0;
    while (part + 1 < p.n_parts && p.strip_prefix[part + 1] <= s) ++part;
    const uint64_t local = s - p.strip_prefix[part];
    const uint32_t spb = p.tpb / 128;
    si.part = part;
    si.x = local / spb;
    si.h = local % spb;
    const uint64_t count = p.parts[part].count;
    const uint64_t base = si.x * uint64_t(p.tpb) * p.ipt + 128 * si.h;
    uint64_t nt = 0;
    if (count > base) nt = (count - base + p.tpb - 1) / p.tpb;
    if (nt > p.ipt) nt = p.ipt;
    if (p.probe_tiles && nt > p.probe_tiles) nt = p.probe_tiles;
    si.n_tiles = uint32_t(nt);
    return si;
}

struct __align__(16) StateEntry {
    double score;
    int32_t acc;
    uint32_t i;
};

template <int KP, bool RW, bool PROBE>
__global__ void __launch_bounds__(kThreads, 1) tensor_scan_kernel(TensorParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t w32 = p.w32;
    const uint32_t stage_bytes = KP * 128 * w32 * 4;
    const uint32_t kbytes = w32 * 4 * 8;        // K bytes = 32 * w32 ... per doc (u8 per dim incl. pad)
    const uint32_t n_kb = w32;                  // one 32-byte K block per 32-dim group
    uint8_t* ring = smem;
    uint8_t* bsm = ring + kStages * stage_bytes;                       // [n_kb][n_pad x 32 B] B image
    uint8_t* after_b = bsm + size_t(p.n_pad) * kbytes;
    // state: main = StateEntry[kQPass][128]; probe = float[kQPass][128]
    uint8_t* state_raw = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(after_b) + 15) & ~uintptr_t(15));
    StateEntry* state = reinterpret_cast<StateEntry*>(state_raw);
    float* pmax = reinterpret_cast<float*>(state_raw);
    uint8_t* after_state = state_raw + (PROBE ? sizeof(float) : sizeof(StateEntry)) * kQPass * 128;
    int32_t* thr = reinterpret_cast<int32_t*>(after_state);            // [kQPass] integer thresholds on D
    int32_t* cq_s = thr + kQPass;                                      // [kQPass]
    double* theta_s = reinterpret_cast<double*>(cq_s + kQPass);        // [kQPass]
    double* t2l_s = theta_s + kQPass;                                  // [kQPass]
    float* red = reinterpret_cast<float*>(t2l_s + kQPass);            // [8] warp mag min/max
    uint64_t* bars = reinterpret_cast<uint64_t*>(red + 8);
    uint64_t* full = bars;
    uint64_t* empty = full + kStages;
    uint64_t* a_full = empty + kStages;
    uint64_t* d_empty = a_full + 2;
    uint64_t* mma_done = d_empty + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_done + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t a_cols = 8 * w32;                 // TMEM columns of one A buffer
    const uint32_t d_cols = p.n_pad;                 // TMEM columns of one D buffer
    uint32_t tmem_cols = 32;
    while (tmem_cols < 2 * (a_cols + d_cols)) tmem_cols <<= 1;

    // ---- one-time setup
    for (uint32_t e = threadIdx.x; e < p.n_pad * kbytes / 16; e += blockDim.x)
        reinterpret_cast<uint4*>(bsm)[e] = reinterpret_cast<const uint4*>(p.bimg)[e];
    for (uint32_t q = threadIdx.x; q < kQPass; q += blockDim.x) {
        const bool live = q < p.nq;
        cq_s[q] = live ? p.cq[p.q0 + q] : 0;
        theta_s[q] = (live && !PROBE) ? p.theta[p.q0 + q] : INFINITY;
        t2l_s[q] = (live && !PROBE) ? p.t2l[p.q0 + q] : INFINITY;
    }
    if (threadIdx.x >= 128 && threadIdx.x < 256) {
        const uint32_t l = threadIdx.x - 128;
        for (uint32_t q = 0; q < kQPass; ++q) {
            if (PROBE) pmax[q * 128 + l] = -INFINITY;
            else state[q * 128 + l].i = kEmpty;
        }
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 128);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(a_full + b, 128);
            mbar_init(d_empty + b, 128);
            mbar_init(mma_done + b, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // make the generic-proxy writes of the B image visible to the tensor core
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t a_col0 = 0;               // A buffers at columns [0, 2*a_cols)
    const uint32_t d_col0 = 2 * a_cols;      // D buffers after them

    if (warp == 8) {
        // ===================== producer =====================
        if (lane == 0) {
            uint32_t u = 0;
            for (uint64_t s = blockIdx.x; s < p.n_strips; s += gridDim.x) {
                const StripInfo si = strip_info(p, s);
                const PartDesc& part = p.parts[si.part];
                for (uint32_t i = 0; i < si.n_tiles; ++i, ++u) {
                    const uint32_t st = u % kStages, k = u / kStages;
                    mbar_wait(empty + st, (k & 1) ^ 1);
                    mbar_expect_tx(full + st, stage_bytes);
                    const uint64_t slot0 = si.x * uint64_t(p.tpb) * p.ipt + uint64_t(i) * p.tpb + 128 * si.h;
                    uint8_t* dst = ring + st * stage_bytes;
#pragma unroll
                    for (int t = 0; t < KP; ++t)
                        bulk_g2s(dst + t * 128 * w32 * 4, part.planes + (uint64_t(t) * part.count_pad + slot0) * w32,
                                 128 * w32 * 4, full + st);
                }
            }
        }
    } else if (warp == 9) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            const uint32_t idesc = idesc_i8(128, p.n_pad);
            const uint32_t b_base = smem_u32(bsm);
            uint32_t u = 0;
            for (uint64_t s = blockIdx.x; s < p.n_strips; s += gridDim.x) {
                const StripInfo si = strip_info(p, s);
                for (uint32_t i = 0; i < si.n_tiles; ++i, ++u) {
                    const uint32_t b = u & 1, j = u >> 1;
                    mbar_wait(a_full + b, j & 1);
                    mbar_wait(d_empty + b, (j & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t a_t = tmem_base + a_col0 + b * a_cols;
                    const uint32_t d_t = tmem_base + d_col0 + b * d_cols;
                    for (uint32_t kb = 0; kb < n_kb; ++kb)
                        mma_i8(d_t, a_t + 8 * kb, smem_desc(b_base + kb * p.n_pad * 32), idesc, kb > 0);
                    mma_commit(mma_done + b);
                }
            }
        }
    } else if (warp < 4) {
        // ===================== expanders =====================
        const uint32_t l = threadIdx.x;  // TMEM lane == doc within the 128-doc sub-tile
        const uint32_t lane_base = uint32_t(warp * 32) << 16;
        uint32_t u = 0;
        for (uint64_t s = blockIdx.x; s < p.n_strips; s += gridDim.x) {
            const StripInfo si = strip_info(p, s);
            for (uint32_t i = 0; i < si.n_tiles; ++i, ++u) {
                const uint32_t st = u % kStages, k = u / kStages;
                const uint32_t b = u & 1, j = u >> 1;
                mbar_wait(full + st, k & 1);
                mbar_wait(mma_done + b, (j & 1) ^ 1);  // A[b] no longer read by the MMA of u-2
                tc_fence_after();
                const uint2* src = reinterpret_cast<const uint2*>(ring + st * stage_bytes);
                const uint32_t a_t = tmem_base + lane_base + a_col0 + b * a_cols;
                const uint32_t w64 = w32 / 2;
                for (uint32_t g2 = 0; g2 < w64; ++g2) {
                    uint32_t w0[KP], w1[KP];
#pragma unroll
                    for (int t = 0; t < KP; ++t) {
                        const uint2 v = src[(t * 128 + l) * w64 + g2];
                        w0[t] = v.x;
                        w1[t] = v.y;
                    }
                    uint32_t out[8];
                    Expand<KP, RW>::run(w0, out);
                    tmem_st8(a_t + 16 * g2, out);
                    Expand<KP, RW>::run(w1, out);
                    tmem_st8(a_t + 16 * g2 + 8, out);
                }
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(a_full + b);
                mbar_arrive(empty + st);
            }
        }
    } else if (warp < 8) {
        // ===================== epilogue =====================
        const uint32_t l = threadIdx.x - 128;
        const int ew = warp - 4;
        const uint32_t lane_base = uint32_t(ew * 32) << 16;
        const int L = int(p.L);
        const uint32_t n_chunks = p.n_pad / 16;
        unsigned long long scored = 0, cands = 0;
        uint32_t u = 0;
        for (uint64_t s = blockIdx.x; s < p.n_strips; s += gridDim.x) {
            const StripInfo si = strip_info(p, s);
            const PartDesc& part = p.parts[si.part];
            for (uint32_t i = 0; i < si.n_tiles; ++i, ++u) {
                const uint32_t b = u & 1, j = u >> 1;
                const uint64_t slot = si.x * uint64_t(p.tpb) * p.ipt + uint64_t(i) * p.tpb + 128 * si.h + l;
                const bool valid = slot < part.count;
                const float mag = valid ? __ldg(part.mags + slot) : 1.0f;
                scored += valid ? 1 : 0;
                if (!PROBE) {
                    // per-sub-tile magnitude range -> integer thresholds on D
                    const uint32_t mb = __float_as_uint(mag);
                    const uint32_t mn = __reduce_min_sync(0xffffffffu, valid ? mb : 0x7f800000u);
                    const uint32_t mx = __reduce_max_sync(0xffffffffu, valid ? mb : 0u);
                    if (lane == 0) {
                        red[ew] = __uint_as_float(mn);
                        red[4 + ew] = __uint_as_float(mx);
                    }
                    named_bar(kEpiBar, 128);
                    if (l < kQPass) {
                        const double mnv = fmin(fmin(red[0], red[1]), fmin(red[2], red[3]));
                        const double mxv = fmax(fmax(red[4], red[5]), fmax(red[6], red[7]));
                        const double t = t2l_s[l];
                        int32_t T;
                        if (!(t > -INFINITY)) {
                            T = INT32_MIN;  // no bound: every pair is a candidate
                        } else if (t == INFINITY || !(mxv > 0.0)) {
                            T = INT32_MAX;  // dead query column / no valid doc
                        } else {
                            // acc = D + C >= t * mag is necessary for score >= theta
                            const double bound = t >= 0.0 ? t * mnv * (1.0 - 1e-12) : t * mxv * (1.0 + 1e-12);
                            const double tf = floor(bound) - double(cq_s[l]) - 1.0;
                            T = tf < -2147483647.0 ? INT32_MIN : (tf > 2147483647.0 ? INT32_MAX : int32_t(tf));
                        }
                        thr[l] = T;
                    }
                    named_bar(kEpiBar, 128);
                }
                mbar_wait(mma_done + b, j & 1);
                tc_fence_after();
                const uint32_t d_t = tmem_base + lane_base + d_col0 + b * d_cols;
                for (uint32_t c = 0; c < n_chunks; ++c) {
                    int32_t acc[16];
                    tmem_ld16(d_t + 16 * c, acc);
                    tmem_wait_ld();
                    if (PROBE) {
                        if (valid) {
                            const float scale = __fdiv_rn(ldexpf(1.0f, -L), mag);
#pragma unroll
                            for (int e = 0; e < 16; ++e) {
                                const uint32_t q = 16 * c + e;
                                const float v = float(acc[e] + cq_s[q]) * scale;
                                float* m = pmax + q * 128 + l;
                                if (v > *m) *m = v;
                            }
                        }
                    } else {
                        uint32_t mask = 0;
#pragma unroll
                        for (int e = 0; e < 16; ++e) mask |= uint32_t(acc[e] >= thr[16 * c + e]) << e;
                        if (!valid) mask = 0;
                        if (mask) {
                            cands += __popc(mask);
                            while (mask) {
                                const int e = __ffs(mask) - 1;
                                mask &= mask - 1;
                                const uint32_t q = 16 * c + e;
                                int32_t a = 0;
#pragma unroll
                                for (int k2 = 0; k2 < 16; ++k2)
                                    if (k2 == e) a = acc[k2];
                                const int32_t accq = a + cq_s[q];
                                const double sc = __ddiv_rn(ldexp(double(accq), -L), double(mag));
                                if (!(sc >= theta_s[q])) continue;
                                StateEntry& st = state[q * 128 + l];
                                if (st.i == kEmpty || sc > st.score) {  // strict: earlier slot wins ties
                                    st.score = sc;
                                    st.acc = accq;
                                    st.i = i;
                                }
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(d_empty + b);
            }
            // ---- strip end: emit survivors (main) / top values (probe)
            if (!PROBE) {
                const uint64_t y_base = si.x * uint64_t(p.tpb) * p.ipt + 128 * si.h + l;
                for (uint32_t q = 0; q < p.nq; ++q) {
                    StateEntry& st = state[q * 128 + l];
                    if (st.i == kEmpty) continue;
                    const uint64_t slot = y_base + uint64_t(st.i) * p.tpb;
                    const unsigned long long pos = atomicAdd(p.surv_count + p.q0 + q, 1ull);
                    if (pos < p.surv_cap) {
                        Result r;
                        r.score = st.score;
                        r.id = part.ids[slot];
                        r.acc = st.acc;
                        r.partition = part.ordinal;
                        r.valid = 1;
                        p.surv[uint64_t(p.q0 + q) * p.surv_cap + pos] = r;
                    }
                    st.i = kEmpty;
                }
            } else {
                named_bar(kEpiBar, 128);
                for (uint32_t q = ew; q < p.nq; q += 4) {
                    float v[4];
#pragma unroll
                    for (int k2 = 0; k2 < 4; ++k2) v[k2] = pmax[q * 128 + 32 * k2 + lane];
                    for (int r = 0; r < kProbeTop; ++r) {
                        float best = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
                        float m = best;
                        for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
                        // remove exactly one copy: the lowest lane holding m
                        const unsigned holder = __ballot_sync(0xffffffffu, best == m);
                        if (lane == __ffs(holder) - 1) {
                            bool done = false;
#pragma unroll
                            for (int k2 = 0; k2 < 4; ++k2)
                                if (!done && v[k2] == m) {
                                    v[k2] = -INFINITY;
                                    done = true;
                                }
                        }
                        if (lane == 0) p.probe_out[uint64_t(p.q0 + q) * p.n_strips * kProbeTop + s * kProbeTop + r] = m;
                    }
                }
                named_bar(kEpiBar, 128);
                for (uint32_t q = 0; q < kQPass; ++q) pmax[q * 128 + l] = -INFINITY;
            }
        }
        if (!PROBE) {
            scored *= p.nq;
            for (int off = 16; off > 0; off >>= 1) {
                scored += __shfl_xor_sync(0xffffffffu, scored, off);
                cands += __shfl_xor_sync(0xffffffffu, cands, off);
            }
            if (lane == 0) {
                atomicAdd(p.scored, scored);
                atomicAdd(p.candidates, cands);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
    }
}

// ------------------------------------------------------------ query operand
// natural query words [Q][qp][wpp] -> B image bytes (2*rq_j as s8) in the
// K-major SWIZZLE_NONE core-matrix layout, per 64-query pass:
//   pass P, K block kb, row r (query), k byte: offset = P*passbytes + kb*(n_pad*32)
//     + (r/8)*256 + ((k%32)/16)*128 + (r%8)*16 + k%16
// and C_q (int32).  One CTA per query.
__global__ void prepare_queries_tensor_kernel(const uint64_t* __restrict__ q, uint32_t Q, uint32_t qp, uint32_t kp,
                                              uint32_t dim, uint32_t wpp, uint32_t rw, uint32_t n_pad,
                                              uint8_t* __restrict__ bimg, int32_t* __restrict__ cq) {
    const uint32_t qi = blockIdx.x;
    const uint32_t K = 64 * wpp;
    const uint32_t pass = qi / kQPass, r = qi % kQPass;
    const size_t pass_bytes = size_t(n_pad) * K;
    __shared__ int64_t part[256];
    int64_t sum = 0;
    for (uint32_t k = threadIdx.x; k < K; k += blockDim.x) {
        int32_t rq = 0;
        for (uint32_t s = 0; s < qp; ++s) {
            const int bit = int((q[(uint64_t(qi) * qp + s) * wpp + k / 64] >> (k % 64)) & 1u);
            rq += rw ? (2 * bit - 1) * (1 << (qp - 1 - s)) : (2 * bit - 1);
        }
        sum += rq;
        const uint32_t kb = k / 32, kk = k % 32;
        const size_t off = pass * pass_bytes + size_t(kb) * n_pad * 32 + (r / 8) * 256 + (kk / 16) * 128 + (r % 8) * 16 +
                           kk % 16;
        bimg[off] = uint8_t(int8_t(2 * rq));
    }
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) part[threadIdx.x] += part[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int64_t pad = int64_t(K) - dim;
        const int64_t vmax = rw ? ((int64_t(1) << kp) - 1) : int64_t(kp);
        const int64_t w = rw ? ((int64_t(1) << qp) - 1) * ((int64_t(1) << kp) - 1) : int64_t(qp) * kp;
        cq[qi] = int32_t(-vmax * part[0] - pad * w);
    }
}

// ------------------------------------------------------------ threshold
// theta_q = (n-th largest probe value) lowered by a relative 2^-16 margin
// (probe scores are FP32 approximations with relative error < 2^-20), or -inf
// when fewer than n finite values exist.  One CTA per query; the first
// kThetaCap values suffice (any subset of distinct threads gives a bound).
constexpr uint32_t kThetaCap = 16384;

__global__ void __launch_bounds__(1024) theta_kernel(const float* __restrict__ probe, uint64_t per_query, uint64_t n,
                                                     uint32_t L, double* theta, double* t2l) {
    extern __shared__ uint32_t keys[];  // [kThetaCap] order-preserving float keys (descending sort)
    const uint32_t q = blockIdx.x;
    const uint32_t m = uint32_t(per_query < kThetaCap ? per_query : kThetaCap);
    uint32_t n2 = 1;
    while (n2 < m) n2 <<= 1;
    __shared__ uint32_t finite_count;
    if (threadIdx.x == 0) finite_count = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
        uint32_t key = 0;  // -inf / padding -> smallest
        if (i < m) {
            const float v = probe[uint64_t(q) * per_query + i];
            if (v > -INFINITY) {
                const uint32_t b = __float_as_uint(v);
                key = (b >> 31) ? ~b : (b | 0x80000000u);
                atomicAdd(&finite_count, 1u);
            }
        }
        keys[i] = key;
    }
    __syncthreads();
    for (uint32_t k = 2; k <= n2; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const bool desc = (i & k) == 0;
                    if ((keys[i] < keys[l]) == desc) {
                        const uint32_t t = keys[i];
                        keys[i] = keys[l];
                        keys[l] = t;
                    }
                }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) {
        double th = -INFINITY;
        if (n > 0 && finite_count >= n) {
            const uint32_t k = keys[n - 1];
            const uint32_t b = (k >> 31) ? (k & 0x7fffffffu) : ~k;
            const double v = double(__uint_as_float(b));
            th = v - fabs(v) * 0x1p-16 - 0x1p-60;
        }
        theta[q] = th;
        t2l[q] = ldexp(th, int(L));
    }
}

uint64_t count_strips(const Shape&, const rbe_scan_geometry& g, uint64_t count) {
    const uint64_t per_block = uint64_t(g.threads_per_block) * g.items_per_thread;
    uint64_t blocks = per_block ? (count + per_block - 1) / per_block : 0;
    if (blocks > g.blocks) blocks = g.blocks;
    return blocks * (g.threads_per_block / 128);
}

template <int KP, bool RW, bool PROBE>
void launch_kernel(const TensorParams& tp, size_t smem, int grid, cudaStream_t st) {
    auto k = tensor_scan_kernel<KP, RW, PROBE>;
    RBE_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k<<<grid, kThreads, smem, st>>>(tp);
    RBE_CK(cudaGetLastError());
}

template <bool PROBE>
void dispatch(uint32_t kp, bool rw, const TensorParams& tp, size_t smem, int grid, cudaStream_t st) {
#define RBE_CASE(K)                                                          \
    case K:                                                                  \
        if (rw) launch_kernel<K, true, PROBE>(tp, smem, grid, st);           \
        else launch_kernel<K, false, PROBE>(tp, smem, grid, st);             \
        return;
    switch (kp) {
        RBE_CASE(1)
        RBE_CASE(2)
        RBE_CASE(3)
        RBE_CASE(4)
        RBE_CASE(5)
        RBE_CASE(6)
        RBE_CASE(7)
        RBE_CASE(8)
        default: throw std::invalid_argument("tensor scan: keyword_planes out of range");
    }
#undef RBE_CASE
}

size_t kernel_smem(uint32_t kp, uint32_t w32, uint32_t n_pad, bool probe) {
    size_t s = size_t(kStages) * kp * 128 * w32 * 4;
    s += size_t(n_pad) * w32 * 32;
    s = (s + 15) & ~size_t(15);
    s += (probe ? 4 : sizeof(StateEntry)) * size_t(kQPass) * 128;
    s += kQPass * 4 * 2 + kQPass * 8 * 2 + 8 * 4;
    s += (kStages * 2 + 6) * 8 + 16;
    return s + 64;
}

int sm_count() {
    int dev = 0, n = 0;
    RBE_CK(cudaGetDevice(&dev));
    RBE_CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

}  // namespace

bool tensor_supported(const Shape& s, uint32_t qp, const rbe_scan_geometry& g, uint32_t Q, std::string* why) {
    auto no = [&](const char* m) {
        if (why) *why = m;
        return false;
    };
    if (g.queue_length != 1) return no("queue_length != 1");
    if (g.threads_per_block % 128 != 0 || g.threads_per_block == 0) return no("threads_per_block not a multiple of 128");
    if (s.kp > 8) return no("more than 8 keyword planes");
    if (s.rw ? qp > 6 : qp > 63) return no("query planes exceed the s8 operand range");
    if (s.wpp > 4) return no("dim > 256");
    if (Q == 0) return no("no queries");
    if (kernel_smem(s.kp, s.w32, kQPass, false) > 227 * 1024) return no("shared memory");
    return true;
}

TensorScanPlan plan_tensor_scan(const Shape& s, uint32_t qp, const rbe_scan_geometry& g, uint32_t Q,
                                const std::vector<uint64_t>& counts, uint64_t n, uint32_t probe_tiles) {
    TensorScanPlan pl;
    pl.Q = Q;
    pl.qp = qp;
    pl.n = n;
    pl.probe_tiles = probe_tiles ? probe_tiles : 8;
    pl.prefix.assign(counts.size() + 1, 0);
    const uint64_t threads = uint64_t(g.blocks) * g.threads_per_block;
    for (size_t i = 0; i < counts.size(); ++i) {
        pl.prefix[i + 1] = pl.prefix[i] + count_strips(s, g, counts[i]);
        pl.surv_cap += std::min<uint64_t>(counts[i], threads);
    }
    pl.surv_cap = std::max<uint64_t>(pl.surv_cap, 1);
    pl.n_strips = pl.prefix.back();
    const uint32_t passes = (Q + kQPass - 1) / kQPass;
    pl.query_bytes = size_t(passes) * kQPass * 64 * s.wpp + size_t(Q) * 4 + 256;
    pl.probe_bytes = size_t(Q) * pl.n_strips * kProbeTop * sizeof(float) + 256;
    pl.threshold_bytes = size_t(Q) * 16 + 64;
    pl.state_bytes = sizeof(uint64_t) * pl.prefix.size() + 64;
    return pl;
}

uint32_t run_tensor_scan(const TensorScanPlan& plan, const ScanArgs& a, const Shape& s, const uint64_t* d_queries,
                         void* d_qtensor, void* d_probe, void* d_thresholds, void* d_state,
                         unsigned long long* d_candidates, cudaStream_t st) {
    const uint32_t Q = a.Q;
    const uint64_t n_strips = plan.n_strips;
    uint64_t* d_prefix = static_cast<uint64_t*>(d_state);
    RBE_CK(cudaMemcpyAsync(d_prefix, plan.prefix.data(), sizeof(uint64_t) * plan.prefix.size(), cudaMemcpyHostToDevice,
                           st));
    const uint32_t passes = (Q + kQPass - 1) / kQPass;
    const uint32_t n_pad = kQPass;
    uint8_t* bimg = static_cast<uint8_t*>(d_qtensor);
    const size_t pass_bytes = size_t(n_pad) * 64 * s.wpp;
    int32_t* cq = reinterpret_cast<int32_t*>(bimg + size_t(passes) * pass_bytes);
    double* theta = static_cast<double*>(d_thresholds);
    double* t2l = theta + Q;
    RBE_CK(cudaMemsetAsync(bimg, 0, size_t(passes) * pass_bytes, st));
    prepare_queries_tensor_kernel<<<Q, 256, 0, st>>>(d_queries, Q, a.qp, s.kp, s.dim, s.wpp, s.rw, n_pad, bimg, cq);
    RBE_CK(cudaGetLastError());
    uint32_t launches = 1;
    const uint64_t per_query = n_strips * kProbeTop;
    float* probe = static_cast<float*>(d_probe);

    TensorParams tp{};
    tp.parts = a.parts;
    tp.strip_prefix = d_prefix;
    tp.n_parts = a.n_parts;
    tp.tpb = a.tpb;
    tp.ipt = a.ipt;
    tp.w32 = s.w32;
    tp.n_pad = n_pad;
    tp.L = s.rw ? (a.qp + s.kp - 2) : 0;
    tp.cq = cq;
    tp.theta = theta;
    tp.t2l = t2l;
    tp.n_strips = n_strips;
    tp.probe_out = probe;
    tp.surv = a.surv;
    tp.surv_count = a.surv_count;
    tp.surv_cap = a.surv_cap;
    tp.scored = a.scored;
    tp.candidates = d_candidates;
    if (n_strips == 0) return launches;
    const int grid = int(std::min<uint64_t>(n_strips, uint64_t(sm_count())));
    for (uint32_t ps = 0; ps < passes; ++ps) {
        tp.q0 = ps * kQPass;
        tp.nq = std::min<uint32_t>(kQPass, Q - tp.q0);
        tp.bimg = bimg + size_t(ps) * pass_bytes;
        // probe pass -> theta
        tp.probe_tiles = plan.probe_tiles;
        dispatch<true>(s.kp, s.rw != 0, tp, kernel_smem(s.kp, s.w32, n_pad, true), grid, st);
        const size_t tsm = size_t(kThetaCap) * 4;
        RBE_CK(cudaFuncSetAttribute(theta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tsm)));
        theta_kernel<<<tp.nq, 1024, tsm, st>>>(probe + uint64_t(tp.q0) * per_query, per_query, plan.n, tp.L,
                                               theta + tp.q0, t2l + tp.q0);
        RBE_CK(cudaGetLastError());
        // main pass
        tp.probe_tiles = 0;
        dispatch<false>(s.kp, s.rw != 0, tp, kernel_smem(s.kp, s.w32, n_pad, false), grid, st);
        launches += 3;
    }
    return launches;
}

}  // namespace rbe_dev
