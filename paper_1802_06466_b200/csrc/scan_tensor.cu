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
// the Expand bit tricks (rbe_common.cuh) straight into TMEM (tcgen05.st),
// which is the MMA's A operand.
//
// Threshold folded into the MMA.  The query operand carries sigma * rq
// (sigma = 2 lambda, a power of two) in the data K blocks plus one extra
// 32-byte K block X whose doc-side bytes are [j, j, j, j, j>>4, 1, 0, 0,
// 255 x 24] with j = the doc's magnitude bin (m >= m0 + Delta j).  The
// tensor core therefore produces, per pair,
//     F = lambda (acc - C_q) + X_q(j),   X_q(j) = c_q - e_q j - g_q (j >> 4),
// with (c, e, g) chosen from the query's current score threshold theta_q so
// that  score >= theta_q  implies  F >= 0  (x_coeffs below; every rounding is
// conservative).  The epilogue only ANDs the 64 accumulators of a doc and
// tests one sign bit; the rare passing pairs recover acc exactly from F and
// are scored in FP64 (IEEE division, bit-identical to the CPU reference).
//
// Selection.  Algorithm 1 keeps, per logical thread (x, y), its best
// queue_length(=1) items (search.cpp:32-48, 57-113); only the top n survivors
// per query matter (search.cpp:115-128, 160-167).  A probe pass over the first
// `probe_tiles` tiles of every logical block gives, per query, the n-th largest
// of per-thread maxima over distinct threads -- a lower bound theta_q on the
// final n-th survivor score.  Items scoring below theta_q can neither be in
// the top n nor change which items >= theta_q survive.  theta_q is raised at
// every strip end from a global histogram of emitted survivors (each a final
// per-thread best of a distinct logical thread), and the X block of the
// query operand is rewritten in shared memory.
//
// Kernel anatomy (one CTA per SM, persistent over "strips" = the sw (256 or
// 128) logical threads [hs*sw, hs*sw + sw) of a logical block; a strip's tile i
// is sw contiguous slots, split into sw/128 sub-tiles of 128 docs):
//   warp 16       producer: cp.async.bulk of each tile's plane words and
//                 magnitudes into a shared-memory ring (mbarrier complete_tx);
//                 TMEM allocator
//   warpgroups    nwg (2..4, four at dim 128) workers; warpgroup w takes
//                 sub-tiles u = w (mod nwg): expand bit planes -> u8 V bytes ->
//                 tcgen05.st into its A (data K blocks; the X block row goes to
//                 shared memory); the last of its four warps to arrive issues the
//                 MMAs into its D (A from TMEM / shared memory, B = queries from
//                 shared memory); the warpgroup then tests D.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "scan_tensor.h"

namespace rbe_dev {
namespace {

constexpr int kStages = 12;          // max ring depth (stages of sw docs)
constexpr int kMaxWG = 4;            // worker warpgroups
// The X (threshold) K block of the doc operand lives in shared memory, not TMEM: TMEM then
// holds per warpgroup two data A operands (8 w32 columns each) and one accumulator, four
// warpgroups at dim 128.  X tile of (warpgroup, A buffer): 128 rows x 16 B (K bytes 0..15,
// core matrices packed, SBO 128); K bytes 16..31 (all 255) come from one shared constant
// tile reached through the descriptor's leading byte offset.
constexpr uint32_t kXTile = 128 * 16;
constexpr int kWGWarps = 4;          // warps per worker warpgroup (4: one per TMEM lane quadrant, 8: two)
constexpr int kHalves = kWGWarps / 4;  // warps sharing each doc (split of its K blocks and queries)
constexpr int kQH = 64 / kHalves;    // accumulator columns (queries) tested per warp
constexpr int kThreads = 32 * (kMaxWG * kWGWarps + 1);  // workers + producer warp
constexpr int kProducerWarp = kMaxWG * kWGWarps;
constexpr uint32_t kCandQueue = 2560;  // deferred candidates per strip (shared memory; overflow is scored at once)
constexpr uint32_t kTouchedCap = 4096;  // state entries listed per strip (beyond: the strip end scans the table)
constexpr int kAllBar = 8;           // named barrier of all worker threads
constexpr int kQPass = 64;           // queries per pass (= MMA N; state is [64][128] in shared memory)
constexpr uint32_t kEmptyKey = ~0u;      // state key: (i << 23) | (acc & 0x7fffff), i < 511, |acc| < 2^22
constexpr uint32_t kThetaCap = 32768;  // probe values per query theta_kernel reads
constexpr int kBins = 64;            // dynamic-theta histogram bins per query
constexpr int kHiCols = 24;          // X block: K bytes 8..31 hold 255 (the c_q "high" part)
constexpr int32_t kXMax = 255 * kHiCols * 127 + 127;  // largest |X| the block can encode
constexpr int32_t kEMax = 4 * 127;   // e_q is split over 4 K bytes
#ifndef RBE_CC_MAXQ
#define RBE_CC_MAXQ 1
#endif
// Small batches (<= kCCMaxQ live queries, dim 128, <= 7 keyword planes): the same kernel scores
// each (doc, query) on the CUDA cores (__dp4a of the expanded doc bytes with the query operand
// rows, plus X_q(j)) instead of the tensor core -- exactly the F the MMA would produce, so the
// candidate sets, the selection and the results are the same; no MMA chain or TMEM round trip
// per sub-tile (the latency path of SURVEY.md C4).
constexpr uint32_t kCCMaxQ = RBE_CC_MAXQ;
constexpr uint32_t kCCUnroll = 8;    // query loop bound of the CUDA-core body (>= kCCMaxQ)
static_assert(kCCMaxQ <= kCCUnroll, "CUDA-core batch bound");

struct TensorParams {
    const PartDesc* parts;
    const uint64_t* strip_prefix;  // [n_parts + 1] cumulative strip counts
    uint32_t n_parts;
    uint32_t tpb, ipt;
    uint32_t w32;                  // u32 words per doc plane (= data K blocks)
    uint32_t nstages;              // ring depth (stages of sw docs)
    uint32_t nwg;                  // worker warpgroups (2 or 3)
    int32_t f16max;                // F <= f16max - c_q for every pair: the low 16 bits keep the sign of any
                                   // F >= 0 when c_q <= 32767 - f16max (pack::16b epilogue); 0 = never
    uint32_t sw;                   // strip width in logical threads (128 or 256) = docs per stage
    uint32_t ptop;                 // probe: values kept per (query, strip)
    uint32_t q0, nq;               // query range of this pass
    uint32_t n_pad;                // MMA N (multiple of 16, >= nq)
    uint32_t L;                    // 2^-L scale (qp + kp - 2, or 0 unweighted)
    uint32_t lam_shift;            // lambda = 2^lam_shift (query operand = 2 lambda rq)
    float m0f, inv_df;             // magnitude bins: j = floor((m - m0) / Delta)
    double m0, delta, mmax;
    const uint8_t* bimg;           // pre-laid-out B image (data K blocks) for this pass
    const int32_t* cq;             // [Q] query constants
    const double* theta;           // [Q] exact-score threshold (main pass)
    uint32_t probe_tiles;          // probe pass: tiles per strip (0 = main pass)
    float* probe_out;              // [Q][n_strips][ptop] (probe launch: n_strips = the probed strips)
    uint64_t n_strips;
    Result* surv;
    unsigned long long* surv_count;
    uint64_t surv_cap;
    unsigned long long* scored;
    unsigned long long* candidates;
    unsigned int* error;
    uint32_t* hist;                // [Q][kBins] emitted-survivor histogram (dynamic theta)
    const double* delta_h;         // [Q] histogram bin width (score units)
    const double* theta0;          // [Q] probe theta (bin 0 lower edge)
    uint64_t n;                    // top-n
    unsigned long long* prof;      // optional [grid][8] phase cycle counters (RBE_PROF=1)
    uint32_t lossless;             // queue_length >= items_per_thread: every item survives its logical
                                   // thread, so pairs >= theta are emitted directly (no per-thread state)
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
// waits on the tensor core: let the hardware suspend the warp until the phase
// completes (or the hint expires) instead of re-polling
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity), "r"(0x100000u)
            : "memory");
    } while (!ok);
}
// waits expected to be long-ish (the tensor core's queue): poll, then nap between polls so a
// waiting warp issues a few instructions instead of waking on every barrier event in the CTA
__device__ __forceinline__ void mbar_wait_nap(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    while (!ok) {
        __nanosleep(64);  // 24 ns measured the same
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
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
// a value the compiler cannot see through (keeps it from hoisting what is cheap to rebuild)
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
    asm volatile("mov.b32 %0, %0;" : "+r"(v));
    return v;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// AND of a predicate over the n worker threads (named barrier kAllBar with .red.and)
__device__ __forceinline__ bool bar_and(bool pred, uint32_t n) {
    uint32_t r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\tbar.red.and.pred q, 8, %2, p;\n\tselp.u32 %0, 1, 0, q;\n}"
        : "=r"(r)
        : "r"(uint32_t(pred)), "r"(n)
        : "memory");
    return r != 0;
}

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
// 64 columns, the low 16 bits of columns 2r and 2r+1 packed into register r
__device__ __forceinline__ void tmem_ld32_p16(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr)
        : "memory");
}
// 32 columns, the low 16 bits of columns 2r and 2r+1 packed into register r
__device__ __forceinline__ void tmem_ld16_p16(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
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
// Executed by a whole warp with warp-uniform operands (kept in uniform registers); one
// elected lane issues.  Issuing from a single divergent lane instead costs ~2x per MMA
// (per-MMA R2UR/ELECT waterfalls: tools/microbench/mma_issue.cu).
__device__ __forceinline__ void mma_i8_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
        : "memory");
}
// one sub-tile: NKB data K blocks + the X block, accumulating into d
// A and B from shared memory (the X block)
__device__ __forceinline__ void mma_i8_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// one sub-tile: NKB data K blocks (A in TMEM) + the X block (A in shared memory), into d
template <int NKB>
__device__ __forceinline__ void mma_group(uint32_t d, uint32_t a, uint64_t b0, uint64_t b_step, uint64_t ax,
                                          uint64_t xd, uint32_t idesc) {
#pragma unroll
    for (int kb = 0; kb < NKB; ++kb) mma_i8_elect(d, a + 8 * kb, b0 + kb * b_step, idesc, kb > 0);
    mma_i8_ss_elect(d, ax, xd, idesc, 1);
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

// same with explicit leading / stride byte offsets
__device__ __forceinline__ uint64_t smem_desc_lbo(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3fffu);
    d |= uint64_t((lbo >> 4) & 0x3fffu) << 16;
    d |= uint64_t((sbo >> 4) & 0x3fffu) << 32;
    d |= uint64_t(1) << 46;
    return d;
}

// instruction descriptor: D s32, A u8 (doc V bytes), B s8 (query 2*rq), K-major both
__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N) {
    return (2u << 4) | (0u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void tmem_st2(uint32_t taddr, uint32_t a, uint32_t b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}

struct StripInfo {
    uint32_t part;
    uint64_t base;     // first slot of the strip: x * tpb * ipt + hs * sw
    uint32_t n_tiles;  // tiles (stages of sw contiguous docs) of the strip
};

// Strip s = logical threads [hs*sw, hs*sw + sw) of logical block x of a partition
// (thread_assignment, search.cpp:10-26): its tile i is the sw contiguous slots
// x*tpb*ipt + i*tpb + hs*sw + [0, sw).
__device__ __forceinline__ StripInfo strip_info(const TensorParams& p, uint64_t s) {
    StripInfo si{0, 0, 0};
    uint32_t part = 0;
    while (part + 1 < p.n_parts && p.strip_prefix[part + 1] <= s) ++part;
    const uint64_t local = s - p.strip_prefix[part];
    const uint32_t spb = p.tpb / p.sw;
    const uint64_t x = local / spb, hs = local % spb;
    si.part = part;
    si.base = x * uint64_t(p.tpb) * p.ipt + p.sw * hs;
    const uint64_t count = p.parts[part].count;
    uint64_t nt = 0;
    if (count > si.base) nt = (count - si.base + p.tpb - 1) / p.tpb;
    if (nt > p.ipt) nt = p.ipt;
    if (p.probe_tiles && nt > p.probe_tiles) nt = p.probe_tiles;
    si.n_tiles = uint32_t(nt);
    return si;
}

// ------------------------------------------------------------ threshold block
struct XCoef {
    int32_t c, e, g;  // X(j) = c - e j - g (j >> 4)
};

// Coefficients of the X block for a query with exact-score threshold theta:
// score >= theta  =>  F = lambda (acc - C_q) + X(j) >= 0 for every doc whose
// magnitude bin is j (m0 + Delta j <= m <= mmax).  score = RN(acc 2^-L / m)
// >= theta implies acc >= t m with t = theta 2^L lowered by 2^-40 relative;
// then X(j) >= lambda (C_q - t m) is required:
//   t >= 0:  lambda (C - t m) <= lambda (C - t m0) - beta j, beta = lambda t Delta,
//            c = ceil(lambda (C - t m0) + margin), e + g/16 <= beta (floors)
//   t <  0:  lambda (C - t m) <= lambda (C - t mmax) = c, e = g = 0.
// Out-of-range values clamp in the conservative direction (larger X).
__device__ XCoef x_coeffs(double theta, int32_t Cq, int L, double lam, double m0, double delta, double mmax) {
    if (!(theta > -INFINITY)) return XCoef{kXMax, 0, 0};  // no bound: every pair passes
    if (theta == INFINITY) return XCoef{-kXMax, 0, 0};    // dead query: no pair passes
    const double t = ldexp(theta, L);
    double c;
    int32_t e = 0, g = 0;
    if (t >= 0.0) {
        const double tl = t * (1.0 - 0x1p-40);
        c = lam * (double(Cq) - tl * m0);
        double beta = lam * tl * delta * (1.0 - 0x1p-40);
        if (beta > double(kEMax)) beta = double(kEMax);
        const double ef = floor(beta);
        e = int32_t(ef);
        g = int32_t(floor((beta - ef) * 16.0 * (1.0 - 0x1p-30)));
        g = g < 0 ? 0 : (g > 15 ? 15 : g);
    } else {
        const double tl = t * (1.0 + 0x1p-40);
        c = lam * (double(Cq) - tl * mmax);
    }
    c = ceil(c + fabs(c) * 0x1p-40 + 1.0);
    if (!(c < double(kXMax))) return XCoef{kXMax, 0, 0};
    if (c < -double(kXMax)) c = -double(kXMax);
    return XCoef{int32_t(c), e, g};
}

// Row r of the X K block (block index kd) of the B image: s8 bytes
// [-e0..-e3, -g, lo, 0, 0, h0..h23], c = 255 sum(h) + lo, e = sum(e_i).
__device__ void write_xrow(uint8_t* bsm, uint32_t n_pad, uint32_t kd, uint32_t r, const XCoef& x) {
    uint8_t* base = bsm + size_t(kd) * n_pad * 32 + (r / 8) * 256 + (r % 8) * 16;
    auto put = [&](int k, int v) { base[(k / 16) * 128 + (k % 16)] = uint8_t(int8_t(v)); };
    const int32_t H = x.c >= 0 ? (x.c + 127) / 255 : -((-x.c + 127) / 255);
    const int32_t lo = x.c - 255 * H;
    for (int i = 0; i < 4; ++i) put(i, -(x.e / 4 + (i < x.e % 4 ? 1 : 0)));
    put(4, -x.g);
    put(5, lo);
    put(6, 0);
    put(7, 0);
    const int32_t hb = H / kHiCols, hr = H - kHiCols * hb;  // hr has the sign of H
    for (int i = 0; i < kHiCols; ++i) {
        int v = hb;
        if (i < (hr >= 0 ? hr : -hr)) v += hr >= 0 ? 1 : -1;
        put(8 + i, v);
    }
}

// magnitude bin: floor((m - m0) / Delta) lowered by 1e-3 so that m0 + Delta j <= m
// holds in real arithmetic despite the float rounding; clamped to [0, 255]
__device__ __forceinline__ uint32_t mag_bin(float m, float m0, float inv_d) {
    float v = __fmaf_rz(m - m0, inv_d, -1.0e-3f);
    v = fminf(fmaxf(v, 0.0f), 255.0f);
    return uint32_t(__float2int_rz(v));
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
    size_t desc, ring, b, xb, state, cqueue, touched, qconst, bars, ax, total;
};

__host__ __device__ inline size_t stage_bytes_of(uint32_t kp, uint32_t w32, uint32_t sw) {
    return size_t(sw) * (size_t(kp) * w32 * 4 + 4);
}

__host__ __device__ inline SmemLayout smem_layout(uint32_t kp, uint32_t w32, uint32_t n_pad, uint32_t nstages,
                                                  uint32_t sw, bool probe) {
    auto al = [](size_t x) { return (x + 127) & ~size_t(127); };
    SmemLayout s{};
    s.desc = 0;  // MMA operand table: [kMaxWG][2 A buffers][2 X parities] x 32 B, at a fixed offset
    const size_t ring = al(kMaxWG * 2 * 2 * 32);
    s.ring = ring;
    size_t off = al(ring + size_t(nstages) * stage_bytes_of(kp, w32, sw));
    s.b = off;  // data K blocks of the query operand
    off = al(off + size_t(n_pad) * 32 * w32);
    s.xb = off;  // two X blocks (threshold), indexed by strip parity
    off = al(off + 2 * size_t(n_pad) * 32);
    s.state = off;  // probe: two [64][sw] float buffers (strip parity)
    off = al(off + size_t(kQPass) * sw * 4 * (probe ? 2 : 1));
    s.cqueue = off;  // also the strip end's histogram / counters scratch
    // (the strip end's counters and histogram, 17 KB, reuse it)
    off = al(off + (probe ? 0 : std::max<size_t>(size_t(kCandQueue) * 8, kQPass * (4 + 8 + 4 * kBins))));
    s.touched = off;
    off = al(off + (probe ? 0 : size_t(kTouchedCap) * 2));
    s.qconst = off;
    off = al(off + kQPass * 8 + kQPass * 4 + 2 * 3 * kQPass * 4 + 16);
    s.bars = off;
    off = al(off + (2 * nstages + 2 * kMaxWG + 2) * 8 + 64);
    s.ax = off;  // [kMaxWG][2] X tiles + the constant tile
    off = al(off + (2 * kMaxWG + 1) * size_t(kXTile));
    s.total = off;
    return s;
}

// One passing pair (F >= 0): score it in FP64 and merge it into the
// per-(query, logical thread) state under (score desc, slot asc)
// (BoundedQueue::insert, search.cpp:32-48).  Entries hold key = (i << 23) |
// (acc & 0x7fffff); the order is independent of insertion order, so threads may
// update the same entry concurrently (CAS).
__device__ __forceinline__ uint32_t key_i(uint32_t key) { return key >> 23; }
__device__ __forceinline__ int32_t key_acc(uint32_t key) { return int32_t(key << 9) >> 9; }
__device__ __noinline__ void take_candidate(int32_t a, uint32_t q, float mag, uint32_t i, uint32_t col, uint32_t sw,
                                            const double* theta_s, uint32_t* st_key, const float* mags_y,
                                            uint32_t tpb, int L, uint16_t* touched, uint32_t* tcount) {
    const double sc = __ddiv_rn(ldexp(double(a), -L), double(mag));
    if (!(sc >= theta_s[q])) return;
    const uint32_t mine = (i << 23) | (uint32_t(a) & 0x7fffffu);
    uint32_t* ent = st_key + q * sw + col;
    uint32_t cur = *ent;
    while (true) {
        if (cur != kEmptyKey) {
            const uint32_t ci = key_i(cur);
            const double cm = double(__ldg(mags_y + uint64_t(ci) * tpb));
            const double cs = __ddiv_rn(ldexp(double(key_acc(cur)), -L), cm);
            if (!(sc > cs || (sc == cs && i < ci))) break;  // the current entry ranks first
        }
        const uint32_t prev = atomicCAS(ent, cur, mine);
        if (prev == cur) {
            if (cur == kEmptyKey) {  // first entry
                const uint32_t pos = atomicAdd(tcount, 1u);
                if (pos < kTouchedCap) touched[pos] = uint16_t(q * sw + col);
            }
            break;
        }
        cur = prev;
    }
}

// A passing pair (F >= 0) of query q and the doc in slot i of logical thread y (mags_y):
// recover acc exactly (F - X(j) = lambda (acc - C_q), j the magnitude bin the X block
// used) and merge it (take_candidate).
__device__ __noinline__ void take_pair(int32_t F, uint32_t q, uint32_t i, uint32_t col, const float* mags_y,
                                       const int32_t* xc, int32_t cq, float m0f, float inv_df, uint32_t lam_shift,
                                       unsigned int* error, uint32_t sw, const double* theta_s, uint32_t* st_key,
                                       uint32_t tpb, int L, uint16_t* touched, uint32_t* tcount) {
    const float mag = __ldg(mags_y + uint64_t(i) * tpb);
    const uint32_t j = mag_bin(mag, m0f, inv_df);
    const int32_t X = xc[q] - xc[kQPass + q] * int32_t(j) - xc[2 * kQPass + q] * int32_t(j >> 4);
    const int32_t num = F - X;
    if (num & ((1 << lam_shift) - 1)) atomicAdd(error, 1u);
    const int32_t a = (num >> lam_shift) + cq;
    take_candidate(a, q, mag, i, col, sw, theta_s, st_key, mags_y, tpb, L, touched, tcount);
}

// Lossless geometry (queue_length >= items_per_thread): BoundedQueue keeps every item of a
// logical thread (search.cpp:32-48), so local_select + global_select reduce to the top n of all
// items under (score desc, id asc).  A passing pair (F >= 0) with its exact score >= theta_q is
// emitted straight into the survivor list; the histogram of emitted (distinct) documents
// refines theta exactly as for per-thread survivors.
__device__ __noinline__ void emit_pair(const TensorParams& p, int32_t F, uint32_t q, uint32_t i, uint32_t col,
                                       const PartDesc& part, uint64_t base, const int32_t* xc, int32_t cq,
                                       const double* theta_s) {
    const uint64_t slot = base + col + uint64_t(i) * p.tpb;
    const float mag = __ldg(part.mags + slot);
    const uint32_t j = mag_bin(mag, p.m0f, p.inv_df);
    const int32_t X = xc[q] - xc[kQPass + q] * int32_t(j) - xc[2 * kQPass + q] * int32_t(j >> 4);
    const int32_t num = F - X;
    if (num & ((1 << p.lam_shift) - 1)) atomicAdd(p.error, 1u);
    const int32_t a = (num >> p.lam_shift) + cq;
    const double sc = __ddiv_rn(ldexp(double(a), -int(p.L)), double(mag));
    if (!(sc >= theta_s[q])) return;
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
    const double dq = p.delta_h[p.q0 + q];
    double fb = floor((sc - p.theta0[p.q0 + q]) / dq);
    fb = fb < 0.0 ? 0.0 : (fb > double(kBins - 1) ? double(kBins - 1) : fb);
    atomicAdd(p.hist + uint64_t(p.q0 + q) * kBins + int(fb), 1u);
}

// Warp roles (17 warps, 120 registers each):
//   warps 0..4*nwg-1   workers: warpgroup w = warp/4 takes sub-tiles u = w (mod nwg)
//                      (128 docs, CTA-local counter u); quadrant warp%4 = TMEM lanes.
//                      Per warpgroup, software-pipelined within a strip:
//                        expand(k+1) -> A[(k+1)&1] while the tensor core runs MMA(k);
//                        wait MMA(k); test D; the last warp of the four to finish issues
//                        MMA(k+1) (A(k+1) ready, D free)
//   warp 16            producer: one contiguous sw-doc stage per tile; TMEM allocator
// phase timing of the worker loop (build with RBE_NVCC_EXTRA=-DRBE_PHASE_PROF, run with RBE_PROF=1)
#ifdef RBE_PHASE_PROF
#define RBE_CLK(x) const long long x = clock64()
#define RBE_ACC(slot, v) prof_acc[slot] += (v)
#else
#define RBE_CLK(x)
#define RBE_ACC(slot, v)
#endif

// W = 4: the common shape fixed at compile time -- dim 128 (w32 = 4), 256-doc strips, three
// worker warpgroups (two in the probe); W = 0: every shape from TensorParams
template <int KP, bool RW, bool PROBE, int W, bool CC = false>
__global__ void __launch_bounds__(kThreads, 1) tensor_scan_kernel(TensorParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr bool kFixed = W == 4;
    const uint32_t w32 = kFixed ? 4u : p.w32;
    const uint32_t nst = p.nstages;
    const uint32_t nwg = kFixed ? 4u : p.nwg;  // 2..4
    const uint32_t n_workers = 32 * kWGWarps * nwg;
    const uint32_t sw = kFixed ? 256u : p.sw;                // strip width (logical threads): 128 or 256
    const uint32_t spt = sw / 128;                           // 128-doc sub-tiles per stage
    const uint32_t spt_sh = spt == 2 ? 1 : 0;
    const uint32_t plane_bytes = sw * w32 * 4;               // one plane of a stage (sw docs)
    const uint32_t stage_bytes = KP * plane_bytes + sw * 4;  // + the stage's f32 magnitudes
    SmemLayout sl = smem_layout(KP, w32, p.n_pad, nst, sw, PROBE);
    uint8_t* ring = smem + sl.ring;
    uint8_t* bsm = smem + sl.b;
    uint8_t* xsm = smem + sl.xb;  // [2][n_pad * 32]
    uint32_t* st_key = reinterpret_cast<uint32_t*>(smem + sl.state);  // [64][sw]
    float* pmax = reinterpret_cast<float*>(smem + sl.state);          // probe: [64][sw]
    uint2* cqueue = reinterpret_cast<uint2*>(smem + sl.cqueue);       // deferred candidates
    uint16_t* touched = reinterpret_cast<uint16_t*>(smem + sl.touched);  // state entries set in the strip
    double* theta_s = reinterpret_cast<double*>(smem + sl.qconst);    // [64]
    int32_t* cq_s = reinterpret_cast<int32_t*>(theta_s + kQPass);     // [64]
    int32_t* xcoef = cq_s + kQPass;                                   // [2][3][64]: c, e, g per strip parity
    uint32_t* p16ok = reinterpret_cast<uint32_t*>(xcoef + 2 * 3 * kQPass);  // [2] packed epilogue safe
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + sl.bars);
    uint64_t* full = bars;                // [nst]   stage loaded (tx bytes)
    uint64_t* empty = full + nst;         // [nst]   stage consumed (4 warp arrivals per sub-tile)
    uint64_t* a_full = empty + nst;       // [kMaxWG] (unused)
    uint64_t* mma_done = a_full + kMaxWG; // [kMaxWG] MMA committed
    uint64_t* x_ready = mma_done + kMaxWG;  // [2] X block of parity b rewritten (strip end)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_ready + 2);
    uint32_t* cq_count = tmem_slot + 1;
    uint32_t* tcount = tmem_slot + 2;
    uint32_t* wg_arrivals = tmem_slot + 4;  // [kMaxWG] per-warpgroup arrival counters (MMA issue)

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t a_cols = 8 * w32;        // TMEM columns of one A (data K blocks, 4 K bytes per column)
    uint8_t* axs = smem + sl.ax;            // X tiles of the doc operand
    const uint32_t d_cols = p.n_pad;        // TMEM columns of one D
    const uint32_t wg_cols = 2 * a_cols + d_cols;
    uint32_t tmem_cols = 32;
    while (tmem_cols < nwg * wg_cols) tmem_cols <<= 1;
    const int L = int(p.L);
    const double lam = double(1u << p.lam_shift);

    // ---- one-time setup: B image (data blocks from global, both X blocks from theta)
    for (uint32_t e = threadIdx.x; e < p.n_pad * 32 * w32 / 16; e += blockDim.x)
        reinterpret_cast<uint4*>(bsm)[e] = reinterpret_cast<const uint4*>(p.bimg)[e];
    for (uint32_t q = threadIdx.x; q < kQPass; q += blockDim.x) {
        const bool live = q < p.nq;
        cq_s[q] = live ? p.cq[p.q0 + q] : 0;
        theta_s[q] = (live && !PROBE) ? p.theta[p.q0 + q] : INFINITY;
        XCoef x;
        if (PROBE) x = live ? XCoef{int32_t(cq_s[q] * int32_t(1u << p.lam_shift)), 0, 0} : XCoef{-kXMax, 0, 0};
        // a padding column (q >= nq) has an all-zero query row, so its F is exactly c: -1 keeps the
        // sign bit of the packed 16-bit epilogue set (c = -kXMax would wrap and flag every doc)
        else x = live ? x_coeffs(theta_s[q], cq_s[q], L, lam, p.m0, p.delta, p.mmax) : XCoef{-1, 0, 0};
        for (int b = 0; b < 2; ++b) {
            xcoef[(b * 3 + 0) * kQPass + q] = x.c;
            xcoef[(b * 3 + 1) * kQPass + q] = x.e;
            xcoef[(b * 3 + 2) * kQPass + q] = x.g;
            write_xrow(xsm + b * p.n_pad * 32, p.n_pad, 0, q, x);
        }
    }
    for (uint32_t e = threadIdx.x; e < kXTile / 4; e += blockDim.x)  // constant X tile: K bytes 16..31 = 255
        reinterpret_cast<uint32_t*>(smem + sl.ax + 2 * kMaxWG * kXTile)[e] = ~0u;
    if (threadIdx.x < 2) p16ok[threadIdx.x] = 1u;
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < p.nq; q += blockDim.x)
        if (p.f16max == 0 || xcoef[q] > 32767 - p.f16max) p16ok[0] = p16ok[1] = 0u;
    for (uint32_t e = threadIdx.x; e < kQPass * sw; e += blockDim.x) {
        if (PROBE) pmax[e] = -INFINITY;
        else st_key[e] = kEmptyKey;
    }
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < nst; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kWGWarps * spt);
        }
        for (int w = 0; w < kMaxWG; ++w) {
            mbar_init(mma_done + w, 1);
        }
        mbar_init(x_ready + 0, 1);
        mbar_init(x_ready + 1, 1);
        *cq_count = 0;
        *tcount = 0;
        for (int w = 0; w < kMaxWG; ++w) wg_arrivals[w] = 0;
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
    // MMA operands of (warpgroup w, A buffer ab, X parity xp), built once: the issuing warp reads
    // 32 bytes instead of rebuilding descriptors on the critical path of every group
    uint4* desc_tab = reinterpret_cast<uint4*>(smem);  // sl.desc == 0
    if (threadIdx.x < kMaxWG * 4) {
        const uint32_t w = threadIdx.x >> 2, ab = (threadIdx.x >> 1) & 1, xp = threadIdx.x & 1;
        const uint64_t b0 = smem_desc(smem_u32(bsm));
        const uint64_t xd = smem_desc(smem_u32(xsm) + xp * p.n_pad * 32);
        const uint64_t axd = smem_desc_lbo(smem_u32(axs) + (w * 2 + ab) * kXTile, (2 * kMaxWG - (w * 2 + ab)) * kXTile, 128);
        const uint32_t a_w = tmem_base + w * wg_cols;
        desc_tab[2 * threadIdx.x] = make_uint4(uint32_t(b0), uint32_t(b0 >> 32), uint32_t(xd), uint32_t(xd >> 32));
        desc_tab[2 * threadIdx.x + 1] = make_uint4(uint32_t(axd), uint32_t(axd >> 32), a_w + ab * a_cols, a_w + 2 * a_cols);
    }
    __syncthreads();

    if (warp == kProducerWarp) {
        // ===================== producer: one contiguous sw-doc stage per tile of each strip =====================
        if (lane == 0) {
            RingPos rs;
            for (uint64_t s = blockIdx.x; s < p.n_strips; s += gridDim.x) {
                const StripInfo si = strip_info(p, s);
                // the partition descriptor in registers (a reference would be re-read from global
                // memory after every bulk copy's memory clobber, serialising the ring on L2 latency)
                const PartDesc part = p.parts[si.part];
                const uint64_t plane_words = part.count_pad * w32;       // u32 words between planes
                const uint32_t* src = part.planes + si.base * w32;       // plane 0 of tile 0
                const float* msrc = part.mags + si.base;
                const uint64_t tile_words = uint64_t(p.tpb) * w32;
                for (uint32_t i = 0; i < si.n_tiles; ++i, rs.next(nst)) {
                    mbar_wait(empty + rs.idx, rs.phase ^ 1);
                    mbar_expect_tx(full + rs.idx, stage_bytes);
                    uint8_t* dst = ring + rs.idx * stage_bytes;
#pragma unroll
                    for (int t = 0; t < KP; ++t)
                        bulk_g2s(dst + t * plane_bytes, src + t * plane_words, plane_bytes, full + rs.idx);
                    bulk_g2s(dst + KP * plane_bytes, msrc, sw * 4, full + rs.idx);
                    src += tile_words;
                    msrc += p.tpb;
                }
            }
        }
    } else if (warp < int(kWGWarps * nwg)) {
        // ===================== workers =====================
        // Warpgroup wg = warps [8 wg, 8 wg + 8).  Warp quadrant warp % 4 owns TMEM lanes
        // (= docs of the sub-tile) [32 quad, 32 quad + 32); the two warps of a quadrant split
        // each doc: half h expands data K blocks [h w32/2, (h+1) w32/2) (half 1 also the X
        // block) and tests accumulator columns (queries) [32h, 32h + 32).
        const uint32_t wg = uint32_t(warp) / kWGWarps;
        const uint32_t half = kHalves == 2 ? (uint32_t(warp) >> 2) & 1u : 0u;
        const int quad = warp & 3;
        const uint32_t l = uint32_t(quad * 32 + lane);  // TMEM lane == doc within the sub-tile
        const uint32_t wt = uint32_t(threadIdx.x);      // worker thread id
        const uint32_t lane_base = uint32_t(quad * 32) << 16;
        const uint32_t hw = w32 / kHalves;              // data K blocks per half
        const uint32_t qh = kQH * half;                 // first query (D column) of this half
        const uint32_t a_t0 = tmem_base + wg * wg_cols + lane_base;  // this warpgroup's A[0] (this warp's lanes)
        const uint32_t d_t = a_t0 + 2 * a_cols + qh;
        const uint32_t pstride = p.ptop;
        uint32_t cands = 0;
        uint32_t kc = 0;  // sub-tiles processed by this warpgroup (A buffer / barrier parities)
#ifdef RBE_PHASE_PROF
        long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // registers: flushed once at the end
#endif
        float pm[PROBE ? kQH : 1];
#pragma unroll
        for (int e = 0; e < (PROBE ? kQH : 1); ++e) pm[e] = -INFINITY;
        // this thread's row (doc l) in its warpgroup's two X tiles: bytes 0..7 per doc, 8..15 = 255
        uint8_t* ax_row = axs + (wg * 2) * kXTile + (l / 8) * 128 + (l % 8) * 16;
        if (half == kHalves - 1) {
            *reinterpret_cast<uint2*>(ax_row + 8) = make_uint2(~0u, ~0u);
            *reinterpret_cast<uint2*>(ax_row + kXTile + 8) = make_uint2(~0u, ~0u);
        }

        // expand this half of doc `col` of ring stage `st` into A buffer `ab`; returns its magnitude
        auto expand = [&](uint32_t st, uint32_t col, uint32_t ab, float& mag) {
            const uint8_t* stage = ring + st * stage_bytes;
            const uint32_t a_t = a_t0 + ab * a_cols;
            if constexpr (W == 4 && kHalves == 1) {
                // one 16-byte load per plane: a warp reads 32 consecutive docs x 16 B, conflict-free
                const uint4* src = reinterpret_cast<const uint4*>(stage) + col;
                uint32_t w0[KP], w1[KP], w2[KP], w3[KP];
#pragma unroll
                for (int t = 0; t < KP; ++t) {
                    const uint4 v = src[t * sw];
                    w0[t] = v.x;
                    w1[t] = v.y;
                    w2[t] = v.z;
                    w3[t] = v.w;
                }
                uint32_t out[16];
                ExpandStored<KP, RW>::run(w0, out);
                ExpandStored<KP, RW>::run(w1, out + 8);
                tmem_st16(a_t, out);
                ExpandStored<KP, RW>::run(w2, out);
                ExpandStored<KP, RW>::run(w3, out + 8);
                tmem_st16(a_t + 16, out);
            } else if constexpr (W == 4) {
                // two 8-byte words per plane: plane t, doc col, words [2h, 2h + 2)
                const uint2* src = reinterpret_cast<const uint2*>(stage) + col * 2 + half;
                uint32_t w0[KP], w1[KP];
#pragma unroll
                for (int t = 0; t < KP; ++t) {
                    const uint2 v = src[t * sw * 2];
                    w0[t] = v.x;
                    w1[t] = v.y;
                }
                uint32_t out[16];
                ExpandStored<KP, RW>::run(w0, out);
                ExpandStored<KP, RW>::run(w1, out + 8);
                tmem_st16(a_t + 16 * half, out);
            } else {
                const uint32_t* src = reinterpret_cast<const uint32_t*>(stage) + col * w32 + hw * half;
                for (uint32_t g = 0; g < hw; ++g) {
                    uint32_t w0[KP];
#pragma unroll
                    for (int t = 0; t < KP; ++t) w0[t] = src[t * sw * w32 + g];
                    uint32_t out[8];
                    ExpandStored<KP, RW>::run(w0, out);
                    tmem_st8(a_t + 8 * (hw * half + g), out);
                }
            }
            mag = reinterpret_cast<const float*>(stage + KP * plane_bytes)[col];
            if (half == kHalves - 1) {
                const uint32_t j = mag_bin(mag, p.m0f, p.inv_df);
                *reinterpret_cast<uint2*>(ax_row + ab * kXTile) = make_uint2(j * 0x01010101u, (j >> 4) | 0x100u);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + st);  // this warp's share of the stage is consumed
        };
        // This warp's part of A(k) is complete and its reads of D are done.  The last of the
        // warpgroup's eight warps to get here issues MMA(k) (whole warp, one elected lane), so no
        // warp ever waits for an issuer: the per-warpgroup counter in shared memory orders it.
        uint32_t xpar = 0;  // X block parity of the current strip
        auto arrive_a = [&](uint32_t ab) {
            tmem_wait_st();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the X row, for the tensor core
            tc_fence_before();
            __syncwarp();
            uint32_t old = 0;
            if (lane == 0)  // acq_rel: publishes this warp's A, acquires the others' for the last arriver
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                             : "=r"(old)
                             : "r"(smem_u32(wg_arrivals + wg))
                             : "memory");
            old = __shfl_sync(0xffffffffu, old, 0);
            if ((old & uint32_t(kWGWarps - 1)) == uint32_t(kWGWarps - 1)) {
                tc_fence_after();
                // MMA N = 64 (run_tensor_scan always pads a pass to kQPass queries): compile-time
                constexpr uint32_t idesc = idesc_i8(128, kQPass);
                constexpr uint64_t b_step = uint64_t(kQPass * 32) >> 4;  // K block stride in descriptor units
                const uint4* e = desc_tab + 2 * (((wg * 2 + ab) * 2) + xpar);
                const uint4 e0 = e[0], e1 = e[1];
                const uint64_t b_desc0 = uint64_t(e0.x) | (uint64_t(e0.y) << 32);
                const uint64_t xd = uint64_t(e0.z) | (uint64_t(e0.w) << 32);
                const uint64_t ax_desc = uint64_t(e1.x) | (uint64_t(e1.y) << 32);
                const uint32_t a_t = e1.z, d_w = e1.w;
                switch (w32) {
                    case 2: mma_group<2>(d_w, a_t, b_desc0, b_step, ax_desc, xd, idesc); break;
                    case 4: mma_group<4>(d_w, a_t, b_desc0, b_step, ax_desc, xd, idesc); break;
                    case 6: mma_group<6>(d_w, a_t, b_desc0, b_step, ax_desc, xd, idesc); break;
                    default: mma_group<8>(d_w, a_t, b_desc0, b_step, ax_desc, xd, idesc); break;
                }
                mma_commit_elect(mma_done + wg);
                __syncwarp();
            }
        };

        uint32_t u0 = 0, tiles0 = 0, sidx = 0;
        for (uint64_t s = blockIdx.x; s < p.n_strips; s += gridDim.x, ++sidx) {
            // only what the sub-tile loop needs stays in registers; the strip's partition and base
            // are recomputed (strip_info) where the rare candidate path and the strip end use them
            uint32_t n_sub, n_tiles, lim;
            {
                const StripInfo si = strip_info(p, s);
                const uint64_t count = p.parts[si.part].count;
                n_tiles = si.n_tiles;
                n_sub = n_tiles * spt;
                // valid: i*tpb + col < lim (i*tpb < 2^31: tensor_supported)
                const uint64_t lim64 = count > si.base ? count - si.base : 0;
                lim = uint32_t(lim64 < 0xffffffffull ? lim64 : 0xffffffffull);
                if (wt == 0 && !PROBE) {
                    // valid docs = sum over tiles t < n_tiles of clamp(lim64 - t tpb, 0, sw), closed form
                    // (sw divides tpb): f full tiles, then at most one partial one
                    const uint64_t f =
                        lim64 >= sw ? std::min<uint64_t>(n_tiles, (lim64 - sw) / p.tpb + 1) : 0;
                    uint64_t valid_docs = f * sw;
                    if (f < n_tiles && lim64 > f * p.tpb) valid_docs += std::min<uint64_t>(lim64 - f * p.tpb, sw);
                    atomicAdd(p.scored, (unsigned long long)(valid_docs * p.nq));
                }
            }
            xpar = sidx & 1;
            // packed-epilogue flag of this strip's X block (fixed for the strip): read once, not
            // on every sub-tile's path from the MMA wait to the accumulator load
            const bool p16 = p16ok[xpar] != 0;
            uint32_t k = (wg + nwg - u0 % nwg) % nwg;
            if constexpr (CC) {
                // ---- CUDA-core body: thread l scores doc l of each of this warpgroup's sub-tiles
                static_assert(W == 4 && KP <= 7, "CUDA-core body: dim 128, u8 doc bytes <= 127 (__dp4a s8)");
                const int32_t* xc = xcoef + xpar * 3 * kQPass;
                const float pscale = PROBE ? ldexpf(1.0f, -L - int(p.lam_shift)) : 0.0f;
                for (; k < n_sub; k += nwg) {
                    const uint32_t ti = k >> spt_sh, t_abs = tiles0 + ti;
                    const uint32_t st_idx = t_abs % nst, st_ph = (t_abs / nst) & 1;
                    const uint32_t col = (k & (spt - 1)) * 128 + l;
                    mbar_wait(full + st_idx, st_ph);
                    const uint8_t* stage = ring + st_idx * stage_bytes;
                    const uint4* src = reinterpret_cast<const uint4*>(stage) + col;
                    uint32_t w0[KP], w1[KP], w2[KP], w3[KP];
#pragma unroll
                    for (int t = 0; t < KP; ++t) {
                        const uint4 v = src[t * sw];
                        w0[t] = v.x;
                        w1[t] = v.y;
                        w2[t] = v.z;
                        w3[t] = v.w;
                    }
                    const float mag = reinterpret_cast<const float*>(stage + KP * plane_bytes)[col];
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + st_idx);
                    uint32_t V[32];  // doc bytes of K [4i, 4i + 4) in V[i] (the A row of the MMA)
                    ExpandStored<KP, RW>::run(w0, V);
                    ExpandStored<KP, RW>::run(w1, V + 8);
                    ExpandStored<KP, RW>::run(w2, V + 16);
                    ExpandStored<KP, RW>::run(w3, V + 24);
                    const int32_t j = int32_t(mag_bin(mag, p.m0f, p.inv_df));
                    const bool valid = ti * p.tpb + col < lim;
                    const float scale = PROBE ? __fdiv_rn(pscale, mag) : 0.0f;
#pragma unroll
                    for (uint32_t q = 0; q < kCCUnroll; ++q) {
                        if (q >= p.nq) break;
                        // F = sum_K V x B_q + X_q(j), B row q of the query operand (core-matrix layout)
                        int32_t F = xc[q] - xc[kQPass + q] * j - xc[2 * kQPass + q] * (j >> 4);
                        const uint8_t* brow = bsm + (q / 8) * 256 + (q % 8) * 16;
#pragma unroll
                        for (int c16 = 0; c16 < 8; ++c16) {
                            const uint4 b = *reinterpret_cast<const uint4*>(brow + (c16 >> 1) * (p.n_pad * 32) +
                                                                            (c16 & 1) * 128);
                            F = __dp4a(int(V[4 * c16 + 0]), int(b.x), F);
                            F = __dp4a(int(V[4 * c16 + 1]), int(b.y), F);
                            F = __dp4a(int(V[4 * c16 + 2]), int(b.z), F);
                            F = __dp4a(int(V[4 * c16 + 3]), int(b.w), F);
                        }
                        if (PROBE) {
                            if (valid) pm[q] = fmaxf(pm[q], float(F) * scale);
                        } else if (F >= 0 && valid) {
                            ++cands;
                            const uint32_t pos = atomicAdd(cq_count, 1u);
                            if (pos < kCandQueue)
                                cqueue[pos] = make_uint2((q << 26) | ti, (col << 24) | uint32_t(F));
                            else {
                                const StripInfo si = strip_info(p, s);
                                if (p.lossless)
                                    emit_pair(p, F, q, ti, col, p.parts[si.part], si.base, xc, cq_s[q], theta_s);
                                else
                                    take_pair(F, q, ti, col, p.parts[si.part].mags + si.base + col, xc, cq_s[q],
                                              p.m0f, p.inv_df, p.lam_shift, p.error, sw, theta_s, st_key, p.tpb, L,
                                              touched, tcount);
                            }
                        }
                    }
                }
            } else if (k < n_sub) {
                // ring position of sub-tile k's stage; advanced incrementally (at most a few stages per step)
                uint32_t ti = k >> spt_sh;
                uint32_t st_idx = (tiles0 + ti) % nst, st_ph = ((tiles0 + ti) / nst) & 1;
                auto seek = [&](uint32_t t_new) {
                    st_idx += t_new - ti;
                    ti = t_new;
                    while (st_idx >= nst) {
                        st_idx -= nst;
                        st_ph ^= 1;
                    }
                };
                float mag, mag_n = 0.0f;
                mbar_wait(full + st_idx, st_ph);
                expand(st_idx, (k & (spt - 1)) * 128 + l, kc & 1, mag);
                arrive_a(kc & 1);
                while (true) {
                    const uint32_t k_n = k + nwg;
                    const bool has_next = k_n < n_sub;
                    const uint32_t i = k >> spt_sh;
                    RBE_CLK(c0);
                    if (has_next) {
                        seek(k_n >> spt_sh);
                        mbar_wait(full + st_idx, st_ph);
                        RBE_CLK(c0b);
                        RBE_ACC(0, c0b - c0);
                        expand(st_idx, (k_n & (spt - 1)) * 128 + l, (kc + 1) & 1, mag_n);
                    }
                    RBE_CLK(c1);
                    const uint32_t col = (k & (spt - 1)) * 128 + l;
                    const bool valid = i * p.tpb + col < lim;
                    mbar_wait_nap(mma_done + wg, kc & 1);
                    tc_fence_after();
                    RBE_CLK(c2);
                    if (PROBE) {
                        // F = lambda acc; per-thread maxima of the (float) score
                        const float scale = __fdiv_rn(ldexpf(1.0f, -L - int(p.lam_shift)), mag);
#pragma unroll
                        for (int c = 0; c < kQH / 16; ++c) {
                            int32_t F[16];
                            tmem_ld16(d_t + 16 * c, F);
                            tmem_wait_ld();
                            if (valid) {
#pragma unroll
                                for (int e2 = 0; e2 < 16; ++e2)
                                    pm[16 * c + e2] = fmaxf(pm[16 * c + e2], float(F[e2]) * scale);
                            }
                        }
                    } else {
                        // F >= 0 is necessary for score >= theta: AND the sign bits per group of 8
                        constexpr int kG = kQH / 8;  // groups of 8 queries per warp
                        uint32_t gmask = 0;  // bit g: some F >= 0 among queries qh + [8g, 8g+8)
                        if (p16) {
                            // low 16 bits of the warp's accumulators, two per register (pack::16b); the
                            // sign of every F >= 0 survives, a wrapped F < 0 is rejected exactly below
                            uint32_t R[kQH / 2];
                            if constexpr (kQH == 64) tmem_ld32_p16(d_t, R);
                            else tmem_ld16_p16(d_t, R);
                            tmem_wait_ld();
                            uint32_t a4[kG];
#pragma unroll
                            for (int g = 0; g < kG; ++g) a4[g] = (R[4 * g] & R[4 * g + 1]) & (R[4 * g + 2] & R[4 * g + 3]);
                            uint32_t all = a4[0];
#pragma unroll
                            for (int g = 1; g < kG; ++g) all &= a4[g];
                            if ((~all & 0x80008000u) && valid) {
#pragma unroll
                                for (int g = 0; g < kG; ++g) gmask |= uint32_t((~a4[g] & 0x80008000u) != 0u) << g;
                            }
                        } else {
#pragma unroll
                            for (int c = 0; c < kQH / 16; ++c) {
                                int32_t F[16];
                                tmem_ld16(d_t + 16 * c, F);
                                tmem_wait_ld();
#pragma unroll
                                for (int g = 0; g < 2; ++g) {
                                    uint32_t a = uint32_t(F[8 * g]);
#pragma unroll
                                    for (int e2 = 1; e2 < 8; ++e2) a &= uint32_t(F[8 * g + e2]);
                                    gmask |= (~a >> 31) << (2 * c + g);
                                }
                            }
                            if (!valid) gmask = 0;
                        }
                        // groups with a passing pair in any lane (tcgen05.ld is warp-collective)
                        // a vote first (short latency; candidates are rare), the OR of the masks only then
                        if (__any_sync(0xffffffffu, gmask != 0u)) {
                            uint32_t wmask = __reduce_or_sync(0xffffffffu, gmask);
                            do {
                                const uint32_t g = uint32_t(__ffs(wmask) - 1);
                                wmask &= wmask - 1;
                                int32_t v[8];
                                tmem_ld8(d_t + 8 * g, v);
                                tmem_wait_ld();
                                if (!((gmask >> g) & 1)) continue;
#pragma unroll
                                for (int e2 = 0; e2 < 8; ++e2) {
                                    if (v[e2] < 0) continue;
                                    ++cands;
                                    const uint32_t q = qh + 8 * g + uint32_t(e2);
                                    // defer to the strip end (acc recovery + exact FP64 scoring in bulk;
                                    // 0 <= F < 2^24); score now if the queue is full
                                    const uint32_t pos = atomicAdd(cq_count, 1u);
                                    if (pos < kCandQueue)
                                        cqueue[pos] = make_uint2((q << 26) | i, (col << 24) | uint32_t(v[e2]));
                                    else {
                                        const StripInfo si = strip_info(p, s);
                                        if (p.lossless)
                                            emit_pair(p, v[e2], q, i, col, p.parts[si.part], si.base,
                                                      xcoef + xpar * 3 * kQPass, cq_s[q], theta_s);
                                        else
                                        take_pair(v[e2], q, i, col, p.parts[si.part].mags + si.base + col,
                                                  xcoef + xpar * 3 * kQPass, cq_s[q], p.m0f, p.inv_df, p.lam_shift,
                                                  p.error, sw, theta_s, st_key, p.tpb, L, touched, tcount);
                                    }
                                }
                            } while (wmask);
                        }
                    }
                    ++kc;
                    RBE_CLK(c3);
                    RBE_ACC(1, c1 - c0);
                    RBE_ACC(2, c2 - c1);
                    RBE_ACC(3, c3 - c2);
                    RBE_ACC(5, 1);
                    if (!has_next) break;
                    RBE_CLK(c6);
                    arrive_a(kc & 1);  // A(k+nwg) ready (kc already advanced), D read
                    RBE_CLK(c7);
                    RBE_ACC(6, c7 - c6);
                    k = k_n;
                    mag = mag_n;
                }
                tc_fence_before();
            }
            u0 += n_sub;
            tiles0 += n_tiles;
            RBE_CLK(c4);
            const StripInfo si = strip_info(p, s);
            const PartDesc& part = p.parts[si.part];
            // ================= strip end (all worker threads) =================
            if (PROBE) {
                // merge the warpgroups' per-lane maxima: the lanes of warpgroup w always hold
                // logical threads (w % spt) * 128 + l when nwg is a multiple of spt; otherwise
                // (spt == 2, nwg == 3) the probe runs with one column per warpgroup (host)
                const uint32_t colp = (wg % spt) * 128 + l;
                // every column is held by exactly one warpgroup (nwg == spt) or by two (nwg == 2 spt:
                // warpgroups w and w + spt)
                const bool owned = nwg == spt || nwg == 2 * spt;
                float* pmx = owned ? pmax + (sidx & 1) * kQPass * sw : pmax;  // double-buffered by strip parity
                if (owned) {
                    // the first holder stores (no reset: every column is rewritten each strip), the
                    // second folds its maxima in; the other parity's buffer is still being read by
                    // warps selecting the previous strip
                    if (wg < spt) {
#pragma unroll
                        for (int e = 0; e < kQH; ++e) {
                            pmx[(qh + e) * sw + colp] = pm[e];
                            pm[e] = -INFINITY;
                        }
                    }
                    named_bar(kAllBar, n_workers);
                    if (wg >= spt) {
#pragma unroll
                        for (int e = 0; e < kQH; ++e) {
                            float* m = pmx + (qh + e) * sw + colp;
                            *m = fmaxf(*m, pm[e]);
                            pm[e] = -INFINITY;
                        }
                    }
                    named_bar(kAllBar, n_workers);
                }
                for (uint32_t w = 0; w < (owned ? 0u : nwg); ++w) {
                    if (w == wg) {
#pragma unroll
                        for (int e = 0; e < kQH; ++e) {
                            float* m = pmax + (qh + e) * sw + colp;
                            *m = fmaxf(*m, pm[e]);
                            pm[e] = -INFINITY;
                        }
                    }
                    named_bar(kAllBar, n_workers);
                }
                // per query, ptop (32 or 16) maxima of disjoint groups of the strip's per-thread
                // maxima (lane-wise over the lane's sw/32 columns, then lane pairs): the n-th largest
                // of maxima over disjoint groups of distinct threads still bounds the final n-th
                // survivor from below (theta_kernel), and no warp-serial selection is needed
                const uint32_t vpl = sw / 32;
                for (uint32_t q = uint32_t(warp); q < p.nq; q += kWGWarps * nwg) {
                    float mx = -INFINITY;
#pragma unroll
                    for (int k2 = 0; k2 < 8; ++k2)
                        if (uint32_t(k2) < vpl) mx = fmaxf(mx, pmx[q * sw + 32 * k2 + lane]);
                    if (pstride == 16) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
                    if (lane < pstride) p.probe_out[(uint64_t(p.q0 + q) * p.n_strips + s) * pstride + lane] = mx;
                }
                if (!owned) {
                    named_bar(kAllBar, n_workers);
                    for (uint32_t k2 = wt; k2 < kQPass * sw; k2 += n_workers) pmax[k2] = -INFINITY;
                    named_bar(kAllBar, n_workers);
                }
                continue;
            }
            named_bar(kAllBar, n_workers);
            // exact FP64 scoring of the strip's deferred candidates
            {
                const uint32_t nc = min(*cq_count, uint32_t(kCandQueue));
                for (uint32_t k2 = wt; k2 < nc; k2 += n_workers) {
                    const uint2 c = cqueue[k2];
                    const uint32_t q = c.x >> 26, ii = c.x & 0x3ffffffu, cc = c.y >> 24;
                    if (p.lossless)
                        emit_pair(p, int32_t(c.y & 0xffffffu), q, ii, cc, part, si.base, xcoef + (sidx & 1) * 3 * kQPass,
                                  cq_s[q], theta_s);
                    else
                    take_pair(int32_t(c.y & 0xffffffu), q, ii, cc, part.mags + si.base + cc,
                              xcoef + (sidx & 1) * 3 * kQPass, cq_s[q], p.m0f, p.inv_df, p.lam_shift, p.error, sw,
                              theta_s, st_key, p.tpb, L, touched, tcount);
                }
            }
            named_bar(kAllBar, n_workers);
            if (wt == 0) *cq_count = 0;
            // emit the strip's survivors >= theta (one per (query, logical thread)) from the
            // list of state entries set in this strip, each with its own slot reservation in the
            // query's survivor list (one pass: the list order is irrelevant, global_select sorts);
            // the histogram is merged in shared memory
            {
                uint32_t* hist_s = reinterpret_cast<uint32_t*>(cqueue);  // [64][kBins]
                // entries to visit: the touched list, or the whole table when it overflowed
                const bool scan_all = *tcount > kTouchedCap;
                const uint32_t nt = scan_all ? kQPass * sw : *tcount;
                for (uint32_t k2 = wt; k2 < kQPass * kBins; k2 += n_workers) hist_s[k2] = 0;
                named_bar(kAllBar, n_workers);
                for (uint32_t k2 = wt; k2 < nt; k2 += n_workers) {
                    const uint32_t ent = scan_all ? k2 : touched[k2];
                    const uint32_t key = st_key[ent];
                    if (key == kEmptyKey) continue;
                    st_key[ent] = kEmptyKey;
                    const uint32_t q = ent / sw, cc = ent % sw;
                    const int32_t a = key_acc(key);
                    const uint64_t slot = si.base + cc + uint64_t(key_i(key)) * p.tpb;
                    const double sc = __ddiv_rn(ldexp(double(a), -L), double(__ldg(part.mags + slot)));
                    if (!(sc >= theta_s[q])) continue;  // theta may have risen since the entry was set
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
                    const double dq = p.delta_h[p.q0 + q];
                    double fb = floor((sc - p.theta0[p.q0 + q]) / dq);
                    fb = fb < 0.0 ? 0.0 : (fb > double(kBins - 1) ? double(kBins - 1) : fb);
                    atomicAdd(hist_s + q * kBins + int(fb), 1u);
                }
                named_bar(kAllBar, n_workers);
                for (uint32_t k2 = wt; k2 < p.nq * kBins; k2 += n_workers)
                    if (hist_s[k2]) atomicAdd(p.hist + uint64_t(p.q0) * kBins + k2, hist_s[k2]);
                if (wt == 0) *tcount = 0;
                named_bar(kAllBar, n_workers);
            }
            // ---- dynamic theta (one thread per query): raise theta_q to the lower edge of the
            // highest histogram bin whose suffix count of emitted survivors reaches n (a valid
            // lower bound on the final n-th survivor score: every emitted survivor is the final
            // per-thread best of a distinct logical thread), then rewrite the X block of parity
            // (sidx+1)&1 for the next strip (no MMA is in flight: the workers issue them and
            // are all here).  theta converges within the first strips; later refreshes are
            // spaced out (a stale X block only means a lower, still valid, threshold).
            if (sidx < 4 || (sidx & 3) == 3) {
                int32_t* xw = xcoef + ((sidx + 1) & 1) * 3 * kQPass;
                uint8_t* xbw = xsm + ((sidx + 1) & 1) * p.n_pad * 32;
                bool ok16 = true;
                if (wt < p.nq) {
                    const uint32_t q = wt;
                    const uint32_t* hp = p.hist + uint64_t(p.q0 + q) * kBins;
                    uint64_t suffix = 0;
                    int B = -1;
                    for (int b0 = kBins - 16; b0 >= 0 && B < 0; b0 -= 16) {
                        uint32_t h[16];
#pragma unroll
                        for (int t = 0; t < 16; ++t) h[t] = __ldcg(hp + b0 + t);
#pragma unroll
                        for (int t = 15; t >= 0; --t) {
                            suffix += h[t];
                            if (B < 0 && suffix >= p.n) B = b0 + t;
                        }
                    }
                    if (B > 0) {
                        const double edge = p.theta0[p.q0 + q] + double(B) * p.delta_h[p.q0 + q];
                        const double th = edge - fabs(edge) * 1e-9 - 0x1p-60;
                        if (th > theta_s[q]) theta_s[q] = th;
                    }
                    const XCoef x = x_coeffs(theta_s[q], cq_s[q], L, lam, p.m0, p.delta, p.mmax);
                    xw[q] = x.c;
                    xw[kQPass + q] = x.e;
                    xw[2 * kQPass + q] = x.g;
                    write_xrow(xbw, p.n_pad, 0, q, x);
                    ok16 = p.f16max != 0 && x.c <= 32767 - p.f16max;
                }
                ok16 = bar_and(ok16, n_workers);
                if (wt == 0) p16ok[(sidx + 1) & 1] = ok16 ? 1u : 0u;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                named_bar(kAllBar, n_workers);
            }
            RBE_CLK(c5);
            RBE_ACC(4, c5 - c4);
        }
#ifdef RBE_PHASE_PROF
        if (p.prof && lane == 0)  // per worker warp: [grid][16][8]
            for (int k2 = 0; k2 < 8; ++k2) p.prof[(uint64_t(blockIdx.x) * 16 + warp) * 8 + k2] += prof_acc[k2];
#endif
        if (!PROBE) {
            unsigned long long cd64 = cands;
            for (int off = 16; off > 0; off >>= 1) cd64 += __shfl_xor_sync(0xffffffffu, cd64, off);
            if (lane == 0 && cd64) atomicAdd(p.candidates, cd64);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kProducerWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
    }
}

// ------------------------------------------------------------ query operand
// natural query words [Q][qp][wpp] -> B image bytes (2 lambda rq_j as s8) of
// the data K blocks in the K-major SWIZZLE_NONE core-matrix layout, per
// 64-query pass:
//   pass P, K block kb, row r (query), k byte: offset = P*passbytes + kb*(n_pad*32)
//     + (r/8)*256 + ((k%32)/16)*128 + (r%8)*16 + k%16
// and C_q (int32).  One CTA per query.
__global__ void prepare_queries_tensor_kernel(const uint64_t* __restrict__ q, uint32_t Q, uint32_t qp, uint32_t kp,
                                              uint32_t dim, uint32_t wpp, uint32_t rw, uint32_t n_pad,
                                              uint32_t lam_shift, uint8_t* __restrict__ bimg,
                                              int32_t* __restrict__ cq) {
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
        bimg[off] = uint8_t(int8_t(rq * (2 << lam_shift)));
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

// strip width: 256 logical threads (one 256-doc contiguous stage per tile, the
// bulk-copy size that reaches full HBM bandwidth) when the block width allows it
uint32_t strip_width(const rbe_scan_geometry& g) { return g.threads_per_block % 256 == 0 ? 256u : 128u; }

uint64_t count_strips(const rbe_scan_geometry& g, uint64_t count) {
    const uint64_t per_block = uint64_t(g.threads_per_block) * g.items_per_thread;
    uint64_t blocks = per_block ? (count + per_block - 1) / per_block : 0;
    if (blocks > g.blocks) blocks = g.blocks;
    return blocks * (g.threads_per_block / strip_width(g));
}

bool cc_body(const TensorParams& tp, uint32_t kp) {
    return tp.w32 == 4 && tp.sw == 256 && tp.nwg == 4u && kp <= 7 && tp.nq <= kCCMaxQ;
}

template <int KP, bool RW, bool PROBE>
void launch_kernel(const TensorParams& tp, size_t smem, int grid, cudaStream_t st) {
    const bool fixed = tp.w32 == 4 && tp.sw == 256 && tp.nwg == 4u;
    auto k = fixed ? tensor_scan_kernel<KP, RW, PROBE, 4> : tensor_scan_kernel<KP, RW, PROBE, 0>;
    if constexpr (KP <= 7)
        if (cc_body(tp, KP)) k = tensor_scan_kernel<KP, RW, PROBE, 4, true>;
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

constexpr size_t kSmemLimit = 227 * 1024;

// TMEM: per warpgroup two A operands (data K = 32 w32 bytes) and one 64-column accumulator
uint32_t pick_nwg(uint32_t w32) {
    for (uint32_t n = kMaxWG; n >= 2; --n)
        if (n * (2 * 8 * w32 + kQPass) <= 512) return n;
    return 0;
}

// ring depth: as many stages (<= kStages) as shared memory allows (the probe keeps two state
// tables, so its ring is shallower)
uint32_t pick_stages(uint32_t kp, uint32_t w32, uint32_t sw, bool probe) {
    for (uint32_t ns = kStages; ns >= 2; --ns)
        if (smem_layout(kp, w32, kQPass, ns, sw, probe).total <= kSmemLimit) return ns;
    return 0;
}

// lambda = 2^shift: the largest with |2 lambda rq| <= 127 and the data part of
// F strictly inside the range the X block can offset (all-pass / none-pass).
// Prefers the largest lambda whose data part leaves room for c_q within int16 (the packed
// 16-bit epilogue, sigma K rqmax vmax <= 28000), else the largest that fits the X block.
int pick_lam_shift(const Shape& s, uint32_t qp) {
    const uint64_t rqmax = s.rw ? ((1ull << qp) - 1) : qp;
    const uint64_t vmax = s.rw ? ((1ull << s.kp) - 1) : s.kp;
    const uint64_t K = 32ull * s.w32;
    for (int pass = 0; pass < 2; ++pass)
        for (int sh = 6; sh >= 0; --sh) {
            const uint64_t sigma = 2ull << sh;
            if (sigma * rqmax > 127 || sigma * rqmax * vmax * K >= uint64_t(kXMax)) continue;
            if (pass == 0 && sigma * rqmax * vmax * K > 28000) continue;
            return sh;
        }
    return -1;
}

rbe_scan_geometry g_of(const ScanArgs& a) {
    rbe_scan_geometry g{};
    g.blocks = a.blocks;
    g.threads_per_block = a.tpb;
    g.items_per_thread = a.ipt;
    g.queue_length = a.ql;
    return g;
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
    if (g.queue_length != 1 && g.queue_length < g.items_per_thread)
        return no("1 < queue_length < items_per_thread (partially lossy queues)");
    if (g.threads_per_block % 128 != 0 || g.threads_per_block == 0) return no("threads_per_block not a multiple of 128");
    if (s.kp > 8) return no("more than 8 keyword planes");
    if (s.rw ? qp > 6 : qp > 63) return no("query planes exceed the s8 operand range");
    if (s.wpp > 4) return no("dim > 256");
    if (Q == 0) return no("no queries");
    if (!pick_nwg(s.w32)) return no("tensor memory");
    if (pick_stages(s.kp, s.w32, strip_width(g), true) == 0 || pick_stages(s.kp, s.w32, strip_width(g), false) == 0)
        return no("shared memory");
    if (pick_lam_shift(s, qp) < 0) return no("accumulator range exceeds the threshold block");
    if (g.items_per_thread >= 511) return no("items_per_thread >= 511 (state key)");
    if (uint64_t(g.items_per_thread) * g.threads_per_block >= (1ull << 31)) return no("logical block span >= 2^31 slots");
    {
        const uint64_t rqmax = s.rw ? ((1ull << qp) - 1) : qp, vmax = s.rw ? ((1ull << s.kp) - 1) : s.kp;
        if (64ull * s.wpp * rqmax * vmax >= (1ull << 22)) return no("accumulator range exceeds the state key");
    }
    return true;
}

TensorScanPlan plan_tensor_scan(const Shape& s, uint32_t qp, const rbe_scan_geometry& g, uint32_t Q,
                                const std::vector<uint64_t>& counts, uint64_t n, uint32_t probe_tiles, uint64_t min_cap) {
    TensorScanPlan pl;
    pl.Q = Q;
    pl.qp = qp;
    pl.n = n;
    pl.probe_tiles = probe_tiles ? probe_tiles : 4;  // 4 of 256 tiles per strip (tools/probe_tiles_sweep.py)
    pl.prefix.assign(counts.size() + 1, 0);
    const uint64_t threads = uint64_t(g.blocks) * g.threads_per_block;
    uint64_t total = 0;
    for (size_t i = 0; i < counts.size(); ++i) {
        pl.prefix[i + 1] = pl.prefix[i] + count_strips(g, counts[i]);
        pl.surv_cap += std::min<uint64_t>(counts[i], threads);
        total += counts[i];
    }
    pl.lossless = g.queue_length > 1;  // tensor_supported: queue_length == 1 or >= items_per_thread
    if (pl.lossless) {
        // every document >= theta is a survivor: a bounded list, grown by the caller on overflow
        pl.surv_cap = std::min<uint64_t>(total, std::max<uint64_t>({min_cap, 8 * n, uint64_t(1) << 16}));
    }
    pl.surv_cap = std::max<uint64_t>(pl.surv_cap, 1);
    pl.n_strips = pl.prefix.back();
    const uint32_t passes = (Q + kQPass - 1) / kQPass;
    pl.query_bytes = size_t(passes) * kQPass * 64 * s.wpp + size_t(Q) * 4 + 256;
    // probe values per (query, strip): 32 lane maxima while all strips' fit theta_kernel's
    // window, else 16 lane-pair maxima
    pl.ptop = pl.n_strips * 32 <= kThetaCap ? 32u : 16u;  // group maxima per (query, strip)
    pl.probe_bytes = size_t(Q) * pl.n_strips * pl.ptop * sizeof(float) + 256;
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
    const uint32_t n_pad = kQPass;  // the kernel's MMA issue assumes N = kQPass
    const int lam_shift = pick_lam_shift(s, a.qp);
    if (lam_shift < 0) throw std::invalid_argument("tensor scan: accumulator range exceeds the threshold block");
    uint8_t* bimg = static_cast<uint8_t*>(d_qtensor);
    const size_t pass_bytes = size_t(n_pad) * 64 * s.wpp;
    int32_t* cq = reinterpret_cast<int32_t*>(bimg + size_t(passes) * pass_bytes);
    double* theta = static_cast<double*>(d_thresholds);
    double* t2l = theta + Q;
    double* theta0 = t2l + Q;
    double* delta_h = theta0 + Q;
    uint32_t* hist = reinterpret_cast<uint32_t*>(delta_h + Q);
    RBE_CK(cudaMemsetAsync(hist, 0, size_t(Q) * kBins * 4, st));
    RBE_CK(cudaMemsetAsync(bimg, 0, size_t(passes) * pass_bytes, st));
    prepare_queries_tensor_kernel<<<Q, 256, 0, st>>>(d_queries, Q, a.qp, s.kp, s.dim, s.wpp, s.rw, n_pad,
                                                     uint32_t(lam_shift), bimg, cq);
    RBE_CK(cudaGetLastError());
    uint32_t launches = 1;
    // theta_kernel reads the first kThetaCap probe values of a query (any subset of distinct
    // threads bounds the n-th survivor): the probe runs only over the strips that feed them
    const uint64_t probe_strips = std::min<uint64_t>(n_strips, kThetaCap / plan.ptop);
    const uint64_t per_query = probe_strips * plan.ptop;  // probe_out: [Q][probe_strips][ptop]
    float* probe = static_cast<float*>(d_probe);

    // magnitude bins: m0 + Delta j <= m for j = floor((m - m0)/Delta - 1e-3) in [0, 255]
    const double m0 = double(a.mag_lo), mmax = double(a.mag_hi);
    double delta = (mmax - m0) / 255.0;
    if (!(delta > 0.0)) delta = std::max(m0, 1e-30) * 0x1p-20;

    TensorParams tp{};
    tp.parts = a.parts;
    tp.strip_prefix = d_prefix;
    tp.n_parts = a.n_parts;
    tp.tpb = a.tpb;
    tp.ipt = a.ipt;
    tp.w32 = s.w32;
    tp.sw = strip_width(g_of(a));
    tp.nwg = pick_nwg(s.w32);
    {
        // D_sigma <= sigma * vmax * K * rqmax; the packed epilogue is used per strip when every live
        // query's c_q keeps that bound + c_q within int16
        const uint64_t rqmax = s.rw ? ((1ull << a.qp) - 1) : a.qp, vmax = s.rw ? ((1ull << s.kp) - 1) : s.kp;
        const uint64_t dmax = (2ull << lam_shift) * vmax * (64ull * s.wpp) * rqmax;
        tp.f16max = dmax < 32767 ? int32_t(dmax) : 0;
    }
    tp.ptop = plan.ptop;
    tp.n_pad = n_pad;
    tp.L = s.rw ? (a.qp + s.kp - 2) : 0;
    tp.lam_shift = uint32_t(lam_shift);
    tp.m0 = m0;
    tp.delta = delta;
    tp.mmax = mmax;
    tp.m0f = a.mag_lo;
    tp.inv_df = float(1.0 / delta);
    tp.cq = cq;
    tp.theta = theta;
    tp.n_strips = n_strips;
    tp.probe_out = probe;
    tp.surv = a.surv;
    tp.surv_count = a.surv_count;
    tp.surv_cap = a.surv_cap;
    tp.scored = a.scored;
    tp.candidates = d_candidates;
    tp.error = a.error;
    tp.hist = hist;
    tp.delta_h = delta_h;
    tp.theta0 = theta0;
    tp.n = plan.n;
    tp.lossless = plan.lossless ? 1u : 0u;
    if (n_strips == 0) return launches;
    const int grid = int(std::min<uint64_t>(n_strips, uint64_t(sm_count())));
#ifdef RBE_PHASE_PROF
    // profiling builds only (RBE_NVCC_EXTRA=-DRBE_PHASE_PROF): per-warp phase cycles, printed per batch
    static unsigned long long* d_prof = nullptr;
    const bool prof = true;
    if (!d_prof) RBE_CK(cudaMalloc(&d_prof, sizeof(unsigned long long) * 2048 * 16 * 8));
#else
    constexpr bool prof = false;
    unsigned long long* d_prof = nullptr;
#endif
    for (uint32_t ps = 0; ps < passes; ++ps) {
        tp.q0 = ps * kQPass;
        tp.nq = std::min<uint32_t>(kQPass, Q - tp.q0);
        tp.bimg = bimg + size_t(ps) * pass_bytes;
        // probe pass -> theta
        tp.probe_tiles = plan.probe_tiles;
        {
            // probe: a warpgroup's lanes must always hold the same logical threads (nwg = spt)
            TensorParams pp = tp;
            if (tp.sw > 128 && tp.nwg % 2) pp.nwg = 2;  // nwg a multiple of spt (4 stays)
            pp.nstages = pick_stages(s.kp, s.w32, tp.sw, true);
            pp.n_strips = probe_strips;
            dispatch<true>(s.kp, s.rw != 0, pp, smem_layout(s.kp, s.w32, n_pad, pp.nstages, tp.sw, true).total, grid, st);
        }
        const size_t tsm = size_t(kThetaCap) * 4;
        RBE_CK(cudaFuncSetAttribute(theta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tsm)));
        theta_kernel<<<tp.nq, 1024, tsm, st>>>(probe + uint64_t(tp.q0) * per_query, per_query, plan.n, tp.L,
                                               theta + tp.q0, t2l + tp.q0, theta0 + tp.q0, delta_h + tp.q0);
        RBE_CK(cudaGetLastError());
        // main pass
        tp.probe_tiles = 0;
        if (prof) {
            RBE_CK(cudaMemsetAsync(d_prof, 0, sizeof(unsigned long long) * 2048 * 16 * 8, st));
            tp.prof = d_prof;
        }
        tp.nstages = pick_stages(s.kp, s.w32, tp.sw, false);
        dispatch<false>(s.kp, s.rw != 0, tp, smem_layout(s.kp, s.w32, n_pad, tp.nstages, tp.sw, false).total, grid, st);
        tp.prof = nullptr;
        if (prof) {
            std::vector<unsigned long long> h(size_t(grid) * 16 * 8);
            RBE_CK(cudaMemcpyAsync(h.data(), d_prof, h.size() * 8, cudaMemcpyDeviceToHost, st));
            RBE_CK(cudaStreamSynchronize(st));
            for (int w = 0; w < 4 * int(tp.nwg); ++w) {
                double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int b = 0; b < grid; ++b)
                    for (int k = 0; k < 8; ++k) acc[k] += double(h[(size_t(b) * 16 + w) * 8 + k]);
                fprintf(stderr, "[rbe prof] warp %2d per sub-tile: wait full %.0f, expand %.0f, wait MMA %.0f, test %.0f, "
                                "arrive+issue %.0f; strip ends %.0f per CTA (n=%.0f)\n",
                        w, acc[0] / acc[5], acc[1] / acc[5], acc[2] / acc[5], acc[3] / acc[5], acc[6] / acc[5],
                        acc[4] / grid, acc[5]);
            }
        }
        launches += 3;
    }
    return launches;
}

}  // namespace rbe_dev
