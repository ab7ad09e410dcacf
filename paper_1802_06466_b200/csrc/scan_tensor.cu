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

constexpr int kStages = 6;           // ring of 128-doc sub-tiles
constexpr int kWG = 3;               // worker warpgroups (expand -> MMA -> filter each)
constexpr int kWorkerWarps = 4 * kWG;
constexpr int kWorkers = 32 * kWorkerWarps;
constexpr int kProducerWarp = kWorkerWarps;
constexpr int kThreads = kWorkers + 32;
constexpr int kAllBar = 8;           // named barrier of all worker threads (1..kWG: per warpgroup)
constexpr int kQPass = 64;           // queries per pass (state is [64][128] in shared memory)
constexpr uint32_t kEmpty = 0xffffffffu;
constexpr unsigned long long kEmptyKey = ~0ull;
constexpr int kProbeTop = 4;         // per-(query, strip) values kept by the probe
constexpr uint32_t kList = 6;        // deferred FP64 candidates per worker thread
constexpr int kBins = 64;            // dynamic-theta histogram bins per query

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
    uint32_t* hist;                // [Q][kBins] emitted-survivor histogram (dynamic theta)
    const double* delta;           // [Q] histogram bin width (score units)
    const double* theta0;          // [Q] probe theta (bin 0 lower edge)
    uint64_t n;                    // top-n
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
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// short waits: try_wait itself suspends the warp for a hardware-defined window
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try(bar, parity)) {
    }
}
// long waits (the producer on a full ring): back off so the spinning warp does
// not steal issue slots from the working ones
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
    if (mbar_try(bar, parity)) return;
    uint32_t ns = 32;
    while (!mbar_try(bar, parity)) {
        __nanosleep(ns);
        ns = ns < 256 ? ns * 2 : 256;
    }
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
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
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

template <int N>
__device__ __forceinline__ void regs_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }
template <int N>
__device__ __forceinline__ void regs_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }

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


// Stage-1 filter coefficients for query q from t = theta * 2^L (rounded
// down): D >= floor(ta * m + tc) is necessary for score >= theta, where m is
// the minimum (t >= 0) or maximum (t < 0) magnitude of the docs tested.
// No bound (t = -inf) -> everything passes; dead column (t = +inf) -> nothing.
__device__ __forceinline__ void set_filter_coeffs(float t, int32_t cq, float* ta, float* tc) {
    if (!(t > -INFINITY)) {
        *ta = 0.0f;
        *tc = -3.0e9f;
    } else if (t == INFINITY) {
        *ta = 0.0f;
        *tc = 3.0e9f;
    } else {
        *ta = t >= 0.0f ? __fmul_rd(t, 0.99999f) : __fmul_rd(t, 1.00001f);
        *tc = __fadd_rd(-float(cq), -2.0f);
    }
}

// position in a ring of n slots + the parity of the current pass over it
struct RingPos {
    uint32_t idx = 0, phase = 0;
    __device__ __forceinline__ void next(uint32_t n) {
        if (++idx == n) {
            idx = 0;
            phase ^= 1;
        }
    }
};

struct SmemLayout {
    size_t b, state, lists, thr, qconst, bars, total;
};

__host__ __device__ inline SmemLayout smem_layout(uint32_t kp, uint32_t w32, uint32_t n_pad, bool probe) {
    auto al = [](size_t x) { return (x + 127) & ~size_t(127); };
    SmemLayout s{};
    size_t off = al(size_t(kStages) * (kp * 128 * w32 * 4 + 512));
    s.b = off;
    off = al(off + size_t(n_pad) * 32 * w32);
    s.state = off;
    off = al(off + (probe ? size_t(kQPass) * 128 * 4 : size_t(kQPass) * 128 * 8));
    s.lists = off;
    off = al(off + (probe ? 0 : size_t(kWorkers) * kList * 12));
    s.thr = off;
    off = al(off + size_t(kWorkerWarps) * kQPass * 4 + kQPass * 4);
    s.qconst = off;
    off = al(off + kQPass * 8 + kQPass * 4 * 3);
    s.bars = off;
    off = al(off + (kStages * 2 + kWG) * 8 + 16);
    s.total = off;
    return s;
}

template <int KP, bool RW, bool PROBE>
__global__ void __launch_bounds__(kThreads, 1) tensor_scan_kernel(TensorParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t w32 = p.w32;
    const uint32_t plane_bytes = 128 * w32 * 4;          // one plane of a 128-doc sub-tile
    const uint32_t stage_bytes = KP * plane_bytes + 512; // + the sub-tile's f32 magnitudes
    const uint32_t kbytes = 32 * w32;                    // K bytes per row (u8 per bit position)
    const uint32_t n_kb = w32;                           // one 32-byte K block per 32-dim group
    SmemLayout sl = smem_layout(KP, w32, p.n_pad, PROBE);
    uint8_t* ring = smem;
    uint8_t* bsm = smem + sl.b;
    unsigned long long* st_key = reinterpret_cast<unsigned long long*>(smem + sl.state);  // [64][128]
    float* pmax = reinterpret_cast<float*>(smem + sl.state);                              // probe: [64][128]
    uint32_t* ls_qi = reinterpret_cast<uint32_t*>(smem + sl.lists);  // [kList][kWorkers]
    int32_t* ls_acc = reinterpret_cast<int32_t*>(ls_qi + kWorkers * kList);
    float* ls_mag = reinterpret_cast<float*>(ls_acc + kWorkers * kList);
    int32_t* T_w = reinterpret_cast<int32_t*>(smem + sl.thr);        // [kWorkerWarps][64]
    int32_t* cq_s = T_w + kWorkerWarps * kQPass;                      // [64]
    double* theta_s = reinterpret_cast<double*>(smem + sl.qconst);   // [64]
    float* t2l_s = reinterpret_cast<float*>(theta_s + kQPass);       // [64]
    float* ta_s = t2l_s + kQPass;                                     // [64] threshold slope
    float* tc_s = ta_s + kQPass;                                      // [64] threshold offset
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + sl.bars);
    uint64_t* full = bars;
    uint64_t* empty = full + kStages;
    uint64_t* mma_done = empty + kStages;  // [kWG]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_done + kWG);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t a_cols = 8 * w32;   // TMEM columns of one sub-tile's A
    const uint32_t d_cols = p.n_pad;   // TMEM columns of one sub-tile's D
    uint32_t tmem_cols = 32;
    while (tmem_cols < kWG * (a_cols + d_cols)) tmem_cols <<= 1;
    const int L = int(p.L);

    // ---- one-time setup
    for (uint32_t e = threadIdx.x; e < p.n_pad * kbytes / 16; e += blockDim.x)
        reinterpret_cast<uint4*>(bsm)[e] = reinterpret_cast<const uint4*>(p.bimg)[e];
    for (uint32_t q = threadIdx.x; q < kQPass; q += blockDim.x) {
        const bool live = q < p.nq;
        cq_s[q] = live ? p.cq[p.q0 + q] : 0;
        theta_s[q] = (live && !PROBE) ? p.theta[p.q0 + q] : INFINITY;
        // float copy of theta*2^L rounded toward -inf (a conservative filter value)
        const double t = (live && !PROBE) ? p.t2l[p.q0 + q] : INFINITY;
        t2l_s[q] = __double2float_rd(t);
        set_filter_coeffs(t2l_s[q], cq_s[q], ta_s + q, tc_s + q);
    }
    for (uint32_t e = threadIdx.x; e < kQPass * 128; e += blockDim.x) {
        if (PROBE) pmax[e] = -INFINITY;
        else st_key[e] = kEmptyKey;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 128);
        }
        for (int w = 0; w < kWG; ++w) mbar_init(mma_done + w, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kProducerWarp) {
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

    if (warp == kProducerWarp) {
        // ===================== producer: bulk copies of sub-tiles into the ring =====================
        if (lane == 0) {
            RingPos rs;
            for (uint64_t s = blockIdx.x; s < p.n_strips; s += gridDim.x) {
                const StripInfo si = strip_info(p, s);
                const PartDesc& part = p.parts[si.part];
                for (uint32_t i = 0; i < si.n_tiles; ++i, rs.next(kStages)) {
                    mbar_wait_backoff(empty + rs.idx, rs.phase ^ 1);
                    mbar_expect_tx(full + rs.idx, stage_bytes);
                    const uint64_t slot0 = si.x * uint64_t(p.tpb) * p.ipt + uint64_t(i) * p.tpb + 128 * si.h;
                    uint8_t* dst = ring + rs.idx * stage_bytes;
#pragma unroll
                    for (int t = 0; t < KP; ++t)
                        bulk_g2s(dst + t * plane_bytes, part.planes + (uint64_t(t) * part.count_pad + slot0) * w32,
                                 plane_bytes, full + rs.idx);
                    bulk_g2s(dst + KP * plane_bytes, part.mags + slot0, 512, full + rs.idx);
                }
            }
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
        return;
    }

    // ===================== workers: warpgroup wg handles sub-tiles u = wg (mod kWG) =====================
    const uint32_t wg = uint32_t(warp >> 2);
    const int quad = warp & 3;
    const uint32_t l = uint32_t(quad * 32 + lane);        // TMEM lane == doc within the sub-tile
    const uint32_t wt = uint32_t(threadIdx.x);            // worker thread id (list owner)
    const uint32_t lane_base = uint32_t(quad * 32) << 16;
    const uint32_t a_t0 = tmem_base + wg * (a_cols + d_cols);  // this warpgroup's A (lane 0)
    const uint32_t d_t0 = a_t0 + a_cols;                       // and D
    const uint32_t w64 = w32 / 2;
    int32_t* Tme = T_w + warp * kQPass;
    unsigned long long scored = 0, cands = 0;
    uint32_t n_list = 0, mma_phase = 0;
    float pm[PROBE ? kQPass : 1];
#pragma unroll
    for (int e = 0; e < (PROBE ? kQPass : 1); ++e) pm[e] = -INFINITY;

    // exact FP64 rescoring of this thread's deferred candidates.  State entries
    // (query q, doc lane l) hold key = (i << 32 | acc) of the best item so far;
    // "higher score, then lower slot" is order-independent, so warpgroups may
    // update the same entry in any order (64-bit CAS).
    auto flush = [&](const StripInfo& si, const PartDesc& part) {
        const uint64_t y_base = si.x * uint64_t(p.tpb) * p.ipt + 128 * si.h + l;
        for (uint32_t k = 0; k < n_list; ++k) {
            const uint32_t qi = ls_qi[k * kWorkers + wt];
            const uint32_t q = qi >> 26, ii = qi & 0x3ffffffu;
            const int32_t a = ls_acc[k * kWorkers + wt];
            const double sc = __ddiv_rn(ldexp(double(a), -L), double(ls_mag[k * kWorkers + wt]));
            if (!(sc >= theta_s[q])) continue;
            const unsigned long long mine = (uint64_t(ii) << 32) | uint32_t(a);
            unsigned long long* ent = st_key + q * 128 + l;
            unsigned long long cur = *ent;
            while (true) {
                if (cur != kEmptyKey) {
                    const uint32_t ci = uint32_t(cur >> 32);
                    const double cm = double(__ldg(part.mags + y_base + uint64_t(ci) * p.tpb));
                    const double cs = __ddiv_rn(ldexp(double(int32_t(uint32_t(cur))), -L), cm);
                    if (!(sc > cs || (sc == cs && ii < ci))) break;  // current entry ranks first
                }
                const unsigned long long prev = atomicCAS(ent, cur, mine);
                if (prev == cur) break;
                cur = prev;
            }
        }
        n_list = 0;
    };

    uint32_t u0 = 0;  // sub-tiles of earlier strips (this CTA)
    for (uint64_t s = blockIdx.x; s < p.n_strips; s += gridDim.x) {
        const StripInfo si = strip_info(p, s);
        const PartDesc& part = p.parts[si.part];
        // this warpgroup's sub-tiles u = u0 + i with u % kWG == wg
        const uint32_t first = (wg + kWG - u0 % kWG) % kWG;
        for (uint32_t i = first; i < si.n_tiles; i += kWG) {
            const uint32_t u = u0 + i;
            const uint32_t st_idx = u % kStages, st_phase = (u / kStages) & 1;
            mbar_wait(full + st_idx, st_phase);
            const uint8_t* stage = ring + st_idx * stage_bytes;
            // ---- expand this doc into A (u8 V bytes, K-major in TMEM)
            {
                const uint2* src = reinterpret_cast<const uint2*>(stage);
                const uint32_t a_t = a_t0 + lane_base;
                for (uint32_t g2 = 0; g2 < w64; ++g2) {
                    uint32_t w0[KP], w1[KP];
#pragma unroll
                    for (int t = 0; t < KP; ++t) {
                        const uint2 v = src[(t * 128 + l) * w64 + g2];
                        w0[t] = v.x;
                        w1[t] = v.y;
                    }
                    uint32_t out[16];
                    Expand<KP, RW>::run(w0, out);
                    Expand<KP, RW>::run(w1, out + 8);
                    tmem_st16(a_t + 16 * g2, out);
                }
            }
            const uint64_t slot0 = si.x * uint64_t(p.tpb) * p.ipt + uint64_t(i) * p.tpb + 128 * si.h;
            const bool valid = slot0 + l < part.count;
            const float mag = valid ? reinterpret_cast<const float*>(stage + KP * plane_bytes)[l] : 0.0f;
            mbar_arrive(empty + st_idx);  // the ring slot may be refilled
            scored += valid ? 1 : 0;
            if (!PROBE) {
                // this warp's integer thresholds on D (its 32 docs): acc = D + C >= t * mag
                // is necessary for score >= theta (t = theta * 2^L); branch-free
                const uint32_t mb = __float_as_uint(mag);
                const float mn = __uint_as_float(__reduce_min_sync(0xffffffffu, valid ? mb : 0x7f800000u));
                const float mx = __uint_as_float(__reduce_max_sync(0xffffffffu, mb));
#pragma unroll
                for (int hq = 0; hq < 2; ++hq) {
                    const uint32_t tq = uint32_t(lane + 32 * hq);
                    const float ta = ta_s[tq], tc = tc_s[tq];
                    const float v = __fmaf_rd(ta, ta >= 0.0f ? mn : mx, tc);
                    Tme[tq] = __float2int_rd(fminf(fmaxf(v, -2.1e9f), 2.1e9f));
                }
                __syncwarp();
            }
            // ---- the warpgroup's A is complete: one thread issues the MMAs
            tmem_wait_st();
            tc_fence_before();
            named_bar(1 + int(wg), 128);
            if ((threadIdx.x & 127) == 0) {
                tc_fence_after();
                const uint32_t idesc = idesc_i8(128, p.n_pad);
                const uint32_t b_base = smem_u32(bsm);
                for (uint32_t kb = 0; kb < n_kb; ++kb)
                    mma_i8(d_t0, a_t0 + 8 * kb, smem_desc(b_base + kb * p.n_pad * 32), idesc, kb > 0);
                mma_commit(mma_done + wg);
            }
            mbar_wait(mma_done + wg, mma_phase);
            mma_phase ^= 1;
            tc_fence_after();
            const uint32_t d_t = d_t0 + lane_base;
            const float scale = PROBE ? __fdiv_rn(ldexpf(1.0f, -L), mag) : 0.0f;
#pragma unroll
            for (int c = 0; c < kQPass / 32; ++c) {
                int32_t acc[32];
                tmem_ld32(d_t + 32 * c, acc);
                tmem_wait_ld();
                if (PROBE) {
                    if (valid) {
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            pm[32 * c + e] = fmaxf(pm[32 * c + e], float(acc[e] + cq_s[32 * c + e]) * scale);
                    }
                    continue;
                }
                // stage 1: one ISETP per pair against this warp's thresholds,
                // accumulated into one predicate per 16-query group
                bool h0 = false, h1 = false;
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    h0 |= acc[e] >= Tme[32 * c + e];
                    h1 |= acc[16 + e] >= Tme[32 * c + 16 + e];
                }
                uint32_t gm = valid ? (uint32_t(h0) | (uint32_t(h1) << 1)) : 0u;
                const uint32_t any = __reduce_or_sync(0xffffffffu, gm);
                if (!any) continue;
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    if (!(any & (1u << g))) continue;
                    uint32_t mask = 0;
                    if (gm & (1u << g)) {
#pragma unroll
                        for (int e = 0; e < 16; ++e) mask |= uint32_t(acc[16 * g + e] >= Tme[32 * c + 16 * g + e]) << e;
                    }
                    while (mask) {
                        const int e = __ffs(mask) - 1;
                        mask &= mask - 1;
                        int32_t a = 0;
#pragma unroll
                        for (int k2 = 0; k2 < 16; ++k2)
                            if (k2 == e) a = acc[16 * g + k2];
                        const uint32_t q = uint32_t(32 * c + 16 * g + e);
                        const int32_t accq = a + cq_s[q];
                        // stage 2: per-doc float test (conservative), before any FP64 work
                        const float t = t2l_s[q];
                        const float need = t >= 0.0f ? __fmul_rd(__fmul_rd(t, mag), 0.99999f)
                                                     : __fmul_rd(__fmul_rd(t, mag), 1.00001f);
                        if (t > -INFINITY && float(accq) < need - 2.0f) continue;
                        ++cands;
                        if (n_list == kList) flush(si, part);
                        ls_qi[n_list * kWorkers + wt] = (q << 26) | i;
                        ls_acc[n_list * kWorkers + wt] = accq;
                        ls_mag[n_list * kWorkers + wt] = mag;
                        ++n_list;
                    }
                }
            }
            tc_fence_before();  // our D reads are complete before the next MMA into D
        }
        u0 += si.n_tiles;
        // ================= strip end (all worker warps) =================
        if (PROBE) {
            // merge the warpgroups' per-lane maxima, then per query keep the top
            // kProbeTop per-thread maxima of the strip (distinct threads)
            for (uint32_t w = 0; w < uint32_t(kWG); ++w) {
                if (w == wg) {
#pragma unroll
                    for (int e = 0; e < kQPass; ++e) {
                        float* m = pmax + e * 128 + l;
                        *m = fmaxf(*m, pm[e]);
                        pm[e] = -INFINITY;
                    }
                }
                named_bar(kAllBar, kWorkers);
            }
            for (uint32_t q = uint32_t(warp); q < p.nq; q += kWorkerWarps) {
                float v[4];
#pragma unroll
                for (int k2 = 0; k2 < 4; ++k2) v[k2] = pmax[q * 128 + 32 * k2 + lane];
                for (int r = 0; r < kProbeTop; ++r) {
                    const float best = fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3]));
                    float m = best;
                    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
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
            named_bar(kAllBar, kWorkers);
            for (uint32_t e = wt; e < kQPass * 128; e += kWorkers) pmax[e] = -INFINITY;
            named_bar(kAllBar, kWorkers);
            continue;
        }
        flush(si, part);
        named_bar(kAllBar, kWorkers);
        // emit the strip's survivors >= theta (one per (query, logical thread))
        for (uint32_t e = wt; e < p.nq * 128; e += kWorkers) {
            const unsigned long long key = st_key[e];
            if (key == kEmptyKey) continue;
            st_key[e] = kEmptyKey;
            const uint32_t q = e / 128, el = e % 128;
            const uint32_t ii = uint32_t(key >> 32);
            const int32_t a = int32_t(uint32_t(key));
            const uint64_t slot = si.x * uint64_t(p.tpb) * p.ipt + 128 * si.h + el + uint64_t(ii) * p.tpb;
            const double sc = __ddiv_rn(ldexp(double(a), -L), double(__ldg(part.mags + slot)));
            if (!(sc >= theta_s[q])) continue;  // theta may have risen since it was queued
            const unsigned long long pos = atomicAdd(p.surv_count + p.q0 + q, 1ull);
            if (pos < p.surv_cap) {
                Result r;
                r.score = sc;
                r.id = part.ids[slot];
                r.acc = a;
                r.partition = part.ordinal;
                r.valid = 1;
                p.surv[uint64_t(p.q0 + q) * p.surv_cap + pos] = r;
            }
            // every emitted survivor is a final survivor of a distinct logical thread
            const double dq = p.delta[p.q0 + q];
            double fb = floor((sc - p.theta0[p.q0 + q]) / dq);
            fb = fb < 0.0 ? 0.0 : (fb > double(kBins - 1) ? double(kBins - 1) : fb);
            atomicAdd(p.hist + uint64_t(p.q0 + q) * kBins + int(fb), 1u);
        }
        named_bar(kAllBar, kWorkers);
        // ---- dynamic theta: raise theta_q to the lower edge of the highest bin
        // whose suffix count of emitted survivors reaches n (a valid lower bound
        // on the final n-th survivor score).  Worker warp w refreshes q = w (mod 12).
        for (uint32_t q = uint32_t(warp); q < p.nq; q += kWorkerWarps) {
            const uint32_t* hp = p.hist + uint64_t(p.q0 + q) * kBins;
            uint32_t sh = __ldcg(hp + 32 + lane), sl2 = __ldcg(hp + lane);
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t a = __shfl_down_sync(0xffffffffu, sh, off);
                const uint32_t c = __shfl_down_sync(0xffffffffu, sl2, off);
                if (lane + off < 32) {
                    sh += a;
                    sl2 += c;
                }
            }
            const uint32_t tot_hi = __shfl_sync(0xffffffffu, sh, 0);
            sl2 += tot_hi;
            const unsigned mh = __ballot_sync(0xffffffffu, uint64_t(sh) >= p.n);
            const unsigned ml = __ballot_sync(0xffffffffu, uint64_t(sl2) >= p.n);
            int B = -1;
            if (mh) B = 32 + (31 - __clz(mh));
            else if (ml) B = 31 - __clz(ml);
            if (lane == 0 && B > 0) {
                const double edge = p.theta0[p.q0 + q] + double(B) * p.delta[p.q0 + q];
                const double th = edge - fabs(edge) * 1e-9 - 0x1p-60;
                if (th > theta_s[q]) {
                    theta_s[q] = th;
                    const float t = __double2float_rd(ldexp(th, L));
                    t2l_s[q] = t;
                    set_filter_coeffs(t, cq_s[q], ta_s + q, tc_s + q);
                }
            }
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
    tc_fence_before();
    __syncthreads();
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
constexpr uint32_t kThetaCap = 32768;

// theta_q = (n-th largest probe value) lowered by a relative 2^-16 margin
// (probe scores are FP32 approximations with relative error < 2^-20), or -inf
// when fewer than n finite values exist.  One CTA per query: MSD radix select
// (4 x 8-bit digits) over order-preserving u32 keys held in shared memory.
// The first kThetaCap values suffice (any subset of distinct threads bounds).
__global__ void __launch_bounds__(1024) theta_kernel(const float* __restrict__ probe, uint64_t per_query, uint64_t n,
                                                     uint32_t L, double* theta, double* t2l, double* theta0,
                                                     double* delta) {
    extern __shared__ uint32_t keys[];  // [kThetaCap]
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_prefix, s_rank, s_finite, s_maxkey;
    const uint32_t q = blockIdx.x;
    const uint32_t m = uint32_t(per_query < kThetaCap ? per_query : kThetaCap);
    if (threadIdx.x == 0) {
        s_finite = 0;
        s_prefix = 0;
        s_maxkey = 0;
    }
    __syncthreads();
    uint32_t fin = 0, mk = 0;
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const float v = probe[uint64_t(q) * per_query + i];
        uint32_t key = 0;  // -inf -> 0 (never selected when finite_count >= n)
        if (v > -INFINITY) {
            const uint32_t b = __float_as_uint(v);
            key = (b >> 31) ? ~b : (b | 0x80000000u);
            ++fin;
        }
        keys[i] = key;
        mk = max(mk, key);
    }
    atomicAdd(&s_finite, fin);
    atomicMax(&s_maxkey, mk);
    __syncthreads();
    const bool ok = n > 0 && s_finite >= n;
    if (ok) {
        if (threadIdx.x == 0) s_rank = uint32_t(n);  // rank from the top (1-based)
        for (int d = 3; d >= 0; --d) {
            for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
            __syncthreads();
            const uint32_t pre = s_prefix;
            const uint32_t hi_mask = d == 3 ? 0u : (0xffffffffu << (8 * (d + 1)));
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
                const uint32_t k = keys[i];
                if ((k & hi_mask) == pre) atomicAdd(&hist[(k >> (8 * d)) & 0xffu], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t r = s_rank, cum = 0;
                int b = 255;
                for (; b > 0; --b) {
                    if (cum + hist[b] >= r) break;
                    cum += hist[b];
                }
                s_rank = r - cum;
                s_prefix = pre | (uint32_t(b) << (8 * d));
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) {
        double th = -INFINITY;
        if (ok) {
            const uint32_t k = s_prefix;
            const uint32_t b = (k >> 31) ? (k & 0x7fffffffu) : ~k;
            const double v = double(__uint_as_float(b));
            th = v - fabs(v) * 0x1p-16 - 0x1p-60;
        }
        theta[q] = th;
        t2l[q] = ldexp(th, int(L));
        theta0[q] = th;
        // histogram bins for the dynamic refinement span [theta0, max probe value]
        double top = th;
        if (s_maxkey) {
            const uint32_t k = s_maxkey;
            top = double(__uint_as_float((k >> 31) ? (k & 0x7fffffffu) : ~k));
        }
        double d = (top - th) / double(kBins);
        if (!(d > 0.0) || !isfinite(d)) d = fabs(top) * 1e-3 + 1e-30;
        delta[q] = d;
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
    return smem_layout(kp, w32, n_pad, probe).total;
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
    if (g.items_per_thread >= (1u << 26)) return no("items_per_thread >= 2^26");
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
    pl.threshold_bytes = size_t(Q) * (32 + kBins * 4) + 64;
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
    double* theta0 = t2l + Q;
    double* delta = theta0 + Q;
    uint32_t* hist = reinterpret_cast<uint32_t*>(delta + Q);
    RBE_CK(cudaMemsetAsync(hist, 0, size_t(Q) * kBins * 4, st));
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
    tp.hist = hist;
    tp.delta = delta;
    tp.theta0 = theta0;
    tp.n = plan.n;
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
                                               theta + tp.q0, t2l + tp.q0, theta0 + tp.q0, delta + tp.q0);
        RBE_CK(cudaGetLastError());
        // main pass
        tp.probe_tiles = 0;
        dispatch<false>(s.kp, s.rw != 0, tp, kernel_smem(s.kp, s.w32, n_pad, false), grid, st);
        launches += 3;
    }
    return launches;
}

}  // namespace rbe_dev
