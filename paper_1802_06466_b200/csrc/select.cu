// select.cu -- global_select + partition merge (src/search.cpp:115-128,
// 160-167) on the device: the top n survivors per query under entry_less
// (score desc, id asc, search.cpp:50-53).  One CTA per query:
//   * m <= kCap survivors: bitonic sort of the 128-bit keys in shared memory;
//   * otherwise an MSD radix select over the key (8-bit digits, histograms in
//     shared memory) narrows to the boundary bucket, which is then sorted in
//     shared memory; the selected n are sorted in shared memory (or, for
//     n > kCap, with a global-memory bitonic sort inside the same CTA).
// Keys are unique per query (ids are unique), so the result is deterministic
// regardless of the order in which the scan appended survivors.
#include <cuda_runtime.h>

#include "internal.h"

namespace rbe_dev {
namespace {

constexpr int kThreads = 1024;
constexpr uint32_t kCap = 8192;    // keys sorted in shared memory
constexpr uint32_t kSmall = 1024;  // direct sort / radix-select stop size: one key per thread (reg_bitonic)

struct Key {
    uint64_t hi, lo;
};

__device__ __forceinline__ bool key_less(uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl) {
    return ah < bh || (ah == bh && al < bl);
}

__device__ __forceinline__ Key key_of(const Result& r) { return Key{score_desc_key(r.score), r.id}; }

// digit d (0 = most significant) of a 128-bit key
__device__ __forceinline__ uint32_t digit_of(const Key& k, int d) {
    return d < 8 ? uint32_t(k.hi >> (56 - 8 * d)) & 0xffu : uint32_t(k.lo >> (56 - 8 * (d - 8))) & 0xffu;
}

// true if the top `nd` digits of k equal `prefix` (prefix holds nd digits, right-aligned)
__device__ __forceinline__ int cmp_prefix(const Key& k, int nd, uint64_t ph, uint64_t pl) {
    // returns -1 / 0 / +1 comparing the top nd digits of k with the prefix
    if (nd == 0) return 0;
    if (nd <= 8) {
        const uint64_t top = k.hi >> (64 - 8 * nd);
        return top < pl ? -1 : (top > pl ? 1 : 0);
    }
    if (k.hi != ph) return k.hi < ph ? -1 : 1;
    const int ndl = nd - 8;
    const uint64_t top = ndl == 8 ? k.lo : (k.lo >> (64 - 8 * ndl));
    return top < pl ? -1 : (top > pl ? 1 : 0);
}

__device__ void smem_bitonic(uint64_t* kh, uint64_t* kl, uint32_t* ix, uint32_t n2) {
    for (uint32_t k = 2; k <= n2; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const bool gt = key_less(kh[l], kl[l], kh[i], kl[i]);
                    if (gt == up) {
                        uint64_t th = kh[i]; kh[i] = kh[l]; kh[l] = th;
                        uint64_t tl = kl[i]; kl[i] = kl[l]; kl[l] = tl;
                        uint32_t ti = ix[i]; ix[i] = ix[l]; ix[l] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// Bitonic sort of kh/kl/ix[0, n) ascending (n <= blockDim.x = 1024), one key per thread:
// partner exchanges at distance j < 32 by warp shuffles, larger ones through shared
// memory; the keys beyond n sort last (padded with ~0).  Result written back to kh/kl/ix.
__device__ void reg_bitonic(uint64_t* kh, uint64_t* kl, uint32_t* ix, uint32_t n) {
    const uint32_t t = threadIdx.x;
    uint64_t h = ~0ull, lo = ~0ull;
    uint32_t x = 0xffffffffu;
    if (t < n) {
        h = kh[t];
        lo = kl[t];
        x = ix[t];
    }
    __syncthreads();
    for (uint32_t k = 2; k <= kThreads; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            uint64_t ph, pl;
            uint32_t px;
            if (j >= 32) {
                kh[t] = h;
                kl[t] = lo;
                ix[t] = x;
                __syncthreads();
                ph = kh[t ^ j];
                pl = kl[t ^ j];
                px = ix[t ^ j];
                __syncthreads();
            } else {
                ph = __shfl_xor_sync(0xffffffffu, h, j);
                pl = __shfl_xor_sync(0xffffffffu, lo, j);
                px = __shfl_xor_sync(0xffffffffu, x, j);
            }
            const bool asc = (t & k) == 0;
            const bool lower = (t & j) == 0;
            const bool p_less = key_less(ph, pl, h, lo);
            // the lower slot keeps the smaller key when ascending, the larger otherwise
            const bool take = lower == asc ? p_less : !p_less && (ph != h || pl != lo);
            if (take) {
                h = ph;
                lo = pl;
                x = px;
            }
        }
    }
    kh[t] = h;
    kl[t] = lo;
    ix[t] = x;
    __syncthreads();
}

__device__ void global_bitonic(const Result* in, uint32_t* ix, uint32_t n, uint32_t n2) {
    // pads [n, n2) with UINT32_MAX (sorts last)
    for (uint32_t i = n + threadIdx.x; i < n2; i += blockDim.x) ix[i] = 0xffffffffu;
    __syncthreads();
    for (uint32_t k = 2; k <= n2; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const uint32_t a = ix[i], b = ix[l];
                    bool gt;  // key(b) < key(a)
                    if (a == 0xffffffffu) gt = b != 0xffffffffu;
                    else if (b == 0xffffffffu) gt = false;
                    else {
                        const Key ka = key_of(in[a]), kb = key_of(in[b]);
                        gt = key_less(kb.hi, kb.lo, ka.hi, ka.lo);
                    }
                    if (gt == ((i & k) == 0)) { ix[i] = b; ix[l] = a; }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(kThreads) select_topn_kernel(const Result* __restrict__ in_all,
                                                               const unsigned long long* __restrict__ counts,
                                                               uint64_t cap, uint64_t n, Result* __restrict__ out_all,
                                                               uint32_t* __restrict__ scratch_all) {
    extern __shared__ uint64_t smem[];
    uint64_t* kh = smem;                              // [kCap]
    uint64_t* kl = kh + kCap;                         // [kCap]
    uint32_t* ix = reinterpret_cast<uint32_t*>(kl + kCap);  // [kCap]
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_cnt, s_bkt;
    __shared__ uint64_t s_ph, s_pl;
    __shared__ int s_nd;
    __shared__ uint64_t s_r;

    const uint32_t q = blockIdx.x;
    const Result* in = in_all + uint64_t(q) * cap;
    Result* out = out_all + uint64_t(q) * n;
    uint64_t m = counts[q];
    if (m > cap) m = cap;
    const uint64_t n_eff = m < n ? m : n;

    // invalid tail
    for (uint64_t k = n_eff + threadIdx.x; k < n; k += blockDim.x) {
        Result r{};
        out[k] = r;
    }
    if (n_eff == 0) return;

    if (m <= kSmall) {
        for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
            const Key k = key_of(in[i]);
            kh[i] = k.hi; kl[i] = k.lo; ix[i] = i;
        }
        __syncthreads();
        reg_bitonic(kh, kl, ix, uint32_t(m));
        for (uint64_t k = threadIdx.x; k < n_eff; k += blockDim.x) out[k] = in[ix[k]];
        return;
    }

    // ---- radix select of the n_eff-th smallest key
    if (threadIdx.x == 0) { s_ph = 0; s_pl = 0; s_nd = 0; s_r = n_eff; }
    __syncthreads();
    for (int d = 0; d < 16; ++d) {
        for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        const int nd = s_nd;
        const uint64_t ph = s_ph, pl = s_pl;
        for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) {
            const Key k = key_of(in[i]);
            if (cmp_prefix(k, nd, ph, pl) == 0) atomicAdd(&hist[digit_of(k, d)], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t r = s_r, cum = 0;
            uint32_t b = 0;
            for (; b < 256; ++b) {
                if (cum + hist[b] >= r) break;
                cum += hist[b];
            }
            s_r = r - cum;
            s_bkt = hist[b];
            if (d < 8) s_pl = (s_pl << 8) | b;
            else if (d == 8) { s_ph = s_pl; s_pl = b; }
            else s_pl = (s_pl << 8) | b;
            s_nd = d + 1;
        }
        __syncthreads();
        if (s_bkt <= kSmall) break;
    }
    const int nd = s_nd;
    const uint64_t ph = s_ph, pl = s_pl, r = s_r;
    // below-bucket entries are all selected (n_eff - r of them); bucket entries
    // go to shared memory to pick their r smallest.
    uint64_t nsel2 = 1;
    while (nsel2 < n) nsel2 <<= 1;
    uint32_t* sel = scratch_all + uint64_t(q) * nsel2;  // selected input indices
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    __shared__ uint32_t s_bcnt;
    if (threadIdx.x == 0) s_bcnt = 0;
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) {
        const Key k = key_of(in[i]);
        const int c = cmp_prefix(k, nd, ph, pl);
        if (c < 0) {
            sel[atomicAdd(&s_cnt, 1u)] = uint32_t(i);
        } else if (c == 0) {
            const uint32_t p = atomicAdd(&s_bcnt, 1u);
            kh[p] = k.hi; kl[p] = k.lo; ix[p] = uint32_t(i);
        }
    }
    __syncthreads();
    const uint32_t nb = s_bcnt;
    if (nb <= kThreads) {
        reg_bitonic(kh, kl, ix, nb);
    } else {
        uint32_t n2 = 1;
        while (n2 < nb) n2 <<= 1;
        for (uint32_t i = nb + threadIdx.x; i < n2; i += blockDim.x) { kh[i] = ~0ull; kl[i] = ~0ull; ix[i] = 0xffffffffu; }
        __syncthreads();
        smem_bitonic(kh, kl, ix, n2);
    }
    const uint32_t below = s_cnt;
    for (uint32_t k = threadIdx.x; k < r; k += blockDim.x) sel[below + k] = ix[k];
    __syncthreads();
    // ---- sort the n_eff selected entries
    if (n_eff <= kThreads) {
        for (uint32_t i = threadIdx.x; i < n_eff; i += blockDim.x) {
            const Key k = key_of(in[sel[i]]);
            kh[i] = k.hi; kl[i] = k.lo; ix[i] = sel[i];
        }
        __syncthreads();
        reg_bitonic(kh, kl, ix, uint32_t(n_eff));
        for (uint64_t k = threadIdx.x; k < n_eff; k += blockDim.x) out[k] = in[ix[k]];
    } else if (n_eff <= kCap) {
        uint32_t n3 = 1;
        while (n3 < n_eff) n3 <<= 1;
        for (uint32_t i = threadIdx.x; i < n3; i += blockDim.x) {
            if (i < n_eff) {
                const Key k = key_of(in[sel[i]]);
                kh[i] = k.hi; kl[i] = k.lo; ix[i] = sel[i];
            } else {
                kh[i] = ~0ull; kl[i] = ~0ull; ix[i] = 0xffffffffu;
            }
        }
        __syncthreads();
        smem_bitonic(kh, kl, ix, n3);
        for (uint64_t k = threadIdx.x; k < n_eff; k += blockDim.x) out[k] = in[ix[k]];
    } else {
        uint32_t n3 = 1;
        while (n3 < n_eff) n3 <<= 1;
        global_bitonic(in, sel, uint32_t(n_eff), n3);
        for (uint64_t k = threadIdx.x; k < n_eff; k += blockDim.x) out[k] = in[sel[k]];
    }
}

// Result records [Q][n] -> the caller's structure-of-arrays layout (entries past a
// query's count zeroed, counts = valid prefix length): one thread per entry.
__global__ void results_to_soa_kernel(const Result* __restrict__ in, uint32_t Q, uint64_t n, double* __restrict__ S,
                                      uint64_t* __restrict__ I, uint32_t* __restrict__ P, int64_t* __restrict__ A,
                                      uint64_t* __restrict__ C) {
    const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= uint64_t(Q) * n) return;
    const Result r = in[e];
    const bool v = r.valid != 0;
    S[e] = v ? r.score : 0.0;
    I[e] = v ? r.id : 0;
    P[e] = v ? r.partition : 0;
    if (A) A[e] = v ? r.acc : 0;
    // the valid entries of a query are a prefix: its count is where valid flips
    const uint64_t k = e % n;
    if (v && (k + 1 == n || !in[e + 1].valid)) C[e / n] = k + 1;
    if (k == 0 && !v) C[e / n] = 0;
}

}  // namespace

void launch_results_to_soa(const Result* d_in, uint32_t Q, uint64_t n, double* S, uint64_t* I, uint32_t* P,
                           int64_t* A, uint64_t* C, cudaStream_t st) {
    const uint64_t total = uint64_t(Q) * n;
    if (total == 0) return;
    results_to_soa_kernel<<<unsigned((total + 255) / 256), 256, 0, st>>>(d_in, Q, n, S, I, P, A, C);
    RBE_CK(cudaGetLastError());
}

size_t select_scratch_bytes(uint32_t Q, uint64_t cap, uint64_t n) {
    (void)cap;
    // per query: index list padded to the next power of two of n
    uint64_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    return size_t(Q) * size_t(n2 > n ? n2 : n) * sizeof(uint32_t) + 256;
}

void launch_select_topn(const Result* d_in, const unsigned long long* d_counts, uint64_t cap, uint32_t Q, uint64_t n,
                        Result* d_out, void* d_scratch, size_t scratch_bytes, cudaStream_t st) {
    if (Q == 0 || n == 0) return;
    if (cap >= 0xffffffffull) throw std::invalid_argument("search: survivor list too large");
    uint64_t n2 = 1;
    while (n2 < n) n2 <<= 1;
    if (scratch_bytes < size_t(Q) * size_t(n2) * sizeof(uint32_t))
        throw std::logic_error("select: scratch too small");
    const size_t smem = size_t(kCap) * (8 + 8 + 4);
    RBE_CK(cudaFuncSetAttribute(select_topn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    // the scratch index list per query is n2 long (global bitonic pads to n2)
    select_topn_kernel<<<Q, kThreads, smem, st>>>(d_in, d_counts, cap, n, d_out, static_cast<uint32_t*>(d_scratch));
    RBE_CK(cudaGetLastError());
}

}  // namespace rbe_dev
