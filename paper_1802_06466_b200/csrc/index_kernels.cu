// index_kernels.cu -- building the HBM-resident bit-plane-major store:
// re-packing reference-layout partitions, the on-device synthetic corpus
// generator, magnitude validation.
#include <cuda_runtime.h>

#include "internal.h"

namespace rbe_dev {

PlanePerm derive_plane_permutation(uint32_t kp, bool rw) {
    PlanePerm p{};
    for (uint32_t t = 0; t < kMaxPlanes; ++t)
        for (uint32_t b = 0; b < 32; ++b) p.perm[t][b] = uint8_t(b);
    if (kp == 0 || kp > uint32_t(kMaxTensorPlanes)) return p;  // identity (exact kernel only)
    for (uint32_t t = 0; t < kp; ++t) {
        bool used[32] = {};
        for (uint32_t b = 0; b < 32; ++b) {
            uint32_t w[kMaxTensorPlanes] = {};
            w[t] = 1u << b;
            uint32_t out[8];
            expand32_host(int(kp), rw, w, out);
            int dim = -1, nz = 0;
            uint32_t val = 0;
            for (int o = 0; o < 8; ++o)
                for (int k = 0; k < 4; ++k) {
                    const uint32_t v = (out[o] >> (8 * k)) & 0xffu;
                    if (v) {
                        ++nz;
                        dim = 4 * o + k;
                        val = v;
                    }
                }
            const uint32_t want = rw ? (1u << (kp - 1 - t)) : 1u;
            if (nz != 1 || val != want || used[dim])
                throw std::logic_error("expand32 is not a weighted bijection (internal error)");
            used[dim] = true;
            p.perm[t][b] = uint8_t(dim);
        }
    }
    return p;
}

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t n, int threads = kThreads) {
    uint64_t g = (n + threads - 1) / threads;
    if (g > 0x7fffffffull) g = 0x7fffffffull;
    return unsigned(g ? g : 1);
}

__device__ __forceinline__ uint32_t natural_half(const uint64_t* nat, uint64_t doc, uint32_t g, uint32_t wpp) {
    const uint64_t v = nat[doc * wpp + (g >> 1)];
    return (g & 1) ? uint32_t(v >> 32) : uint32_t(v);
}

__device__ __forceinline__ uint32_t permute_word(uint32_t nat, const uint8_t* perm) {
    uint32_t d = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) d |= ((nat >> perm[b]) & 1u) << b;
    return d;
}

__device__ __forceinline__ uint32_t unpermute_word(uint32_t dev, const uint8_t* perm) {
    uint32_t n = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) n |= ((dev >> b) & 1u) << perm[b];
    return n;
}

// natural [kp][count][wpp] u64  ->  device [kp][count_pad][W32] u32 (permuted;
// plane-interleaved for kp = 3 weighted).  One thread per (doc, u32 word).
__global__ void repack_kernel(const uint64_t* __restrict__ nat, uint32_t* __restrict__ dev, uint64_t count,
                              uint64_t count_pad, uint32_t kp, uint32_t wpp, uint32_t rw, PlanePerm perm) {
    const uint32_t w32 = 2 * wpp;
    const uint64_t total = count * w32;
    const bool il = interleaved_store(int(kp), rw != 0);
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t g = uint32_t(e % w32);
        const uint64_t doc = e / w32;
        if (il) {
            uint32_t w[3], z[3];
            for (uint32_t t = 0; t < 3; ++t)
                w[t] = permute_word(natural_half(nat + uint64_t(t) * count * wpp, doc, g, wpp), perm.perm[t]);
            interleave3(w, z);
            for (uint32_t t = 0; t < 3; ++t) dev[(uint64_t(t) * count_pad + doc) * w32 + g] = z[t];
        } else {
            for (uint32_t t = 0; t < kp; ++t) {
                const uint32_t nw = natural_half(nat + uint64_t(t) * count * wpp, doc, g, wpp);
                dev[(uint64_t(t) * count_pad + doc) * w32 + g] = permute_word(nw, perm.perm[t < uint32_t(kMaxPlanes) ? t : 0]);
            }
        }
    }
}

__global__ void unpack_kernel(const uint32_t* __restrict__ dev, uint64_t* __restrict__ nat, uint64_t count,
                              uint64_t count_pad, uint32_t kp, uint32_t wpp, uint32_t rw, PlanePerm perm) {
    const uint64_t total = count * wpp;
    const uint32_t w32 = 2 * wpp;
    const bool il = interleaved_store(int(kp), rw != 0);
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t w = uint32_t(e % wpp);
        const uint64_t doc = e / wpp;
        for (uint32_t t = 0; t < kp; ++t) {
            uint32_t lo, hi;
            if (il) {
                uint32_t z[3], pw[3];
                for (uint32_t c = 0; c < 3; ++c) z[c] = dev[(uint64_t(c) * count_pad + doc) * w32 + 2 * w];
                deinterleave3(z, pw);
                lo = pw[t];
                for (uint32_t c = 0; c < 3; ++c) z[c] = dev[(uint64_t(c) * count_pad + doc) * w32 + 2 * w + 1];
                deinterleave3(z, pw);
                hi = pw[t];
            } else {
                const uint32_t* src = dev + (uint64_t(t) * count_pad + doc) * w32 + 2 * w;
                lo = src[0];
                hi = src[1];
            }
            const uint8_t* pm = perm.perm[t < uint32_t(kMaxPlanes) ? t : 0];
            nat[(uint64_t(t) * count + doc) * wpp + w] = uint64_t(unpermute_word(lo, pm)) | (uint64_t(unpermute_word(hi, pm)) << 32);
        }
    }
}

// One thread per slot of the partition: generate the doc's plane words from
// the counter-based stream, write them permuted, and compute its magnitude by
// replaying refined_vector + make_embedding (src/embedding.cpp:7-36) in the
// same IEEE double operation order (explicit _rn intrinsics: no FMA
// contraction), so float(magnitude) is bit-identical to the CPU reference.
__global__ void fill_synthetic_kernel(uint32_t* __restrict__ planes, float* __restrict__ mags,
                                      uint64_t* __restrict__ ids, uint64_t count, uint64_t count_pad,
                                      uint32_t ordinal, uint32_t n_parts_total, uint64_t n_total, uint64_t seed,
                                      uint32_t dim, uint32_t kp, uint32_t wpp, uint32_t rw, PlanePerm perm) {
    const uint64_t pad_mask = (dim % 64 == 0) ? ~0ull : ((1ull << (dim % 64)) - 1);
    const uint32_t w32 = 2 * wpp;
    for (uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; s < count;
         s += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t gdoc = s * n_parts_total + ordinal;
        double sq = 0.0;
        for (uint32_t w = 0; w < wpp; ++w) {
            const uint32_t nbits = (w + 1 == wpp && dim % 64) ? dim % 64 : 64;
            double x[64];
#pragma unroll
            for (int b = 0; b < 64; ++b) x[b] = 0.0;
            for (uint32_t t = 0; t < kp; ++t) {
                uint64_t v = splitmix64_at(seed, (uint64_t(t) * n_total + gdoc) * wpp + w);
                if (w + 1 == wpp) v &= pad_mask;
                uint32_t* dst = planes + (uint64_t(t) * count_pad + s) * w32 + 2 * w;
                const uint8_t* pm = perm.perm[t < uint32_t(kMaxPlanes) ? t : 0];
                dst[0] = permute_word(uint32_t(v), pm);
                dst[1] = permute_word(uint32_t(v >> 32), pm);
                const double wt = rw ? ldexp(1.0, -int(t)) : 1.0;
#pragma unroll
                for (int b = 0; b < 64; ++b) x[b] = __dadd_rn(x[b], ((v >> b) & 1) ? wt : -wt);
            }
            for (uint32_t b = 0; b < nbits; ++b) sq = __dadd_rn(sq, __dmul_rn(x[b], x[b]));
        }
        if (interleaved_store(int(kp), rw != 0)) {
            for (uint32_t g = 0; g < w32; ++g) {
                uint32_t w[3], z[3];
                for (uint32_t t = 0; t < 3; ++t) w[t] = planes[(uint64_t(t) * count_pad + s) * w32 + g];
                interleave3(w, z);
                for (uint32_t t = 0; t < 3; ++t) planes[(uint64_t(t) * count_pad + s) * w32 + g] = z[t];
            }
        }
        mags[s] = __double2float_rn(__dsqrt_rn(sq));
        ids[s] = gdoc;
    }
}

// RBEE records [rec0, rec0 + n) (raw bytes: u64 id, [kp][wpp] u64 plane words, f32 magnitude;
// embedding_io.cpp:32-45, records 4-byte aligned in the file, so words are read as u32 halves)
// -> the store, with IndexBuilder::add's semantics (src/index.cpp:36-78): record k goes to
// partition k % P, slot k / P, if this handle holds that partition (local[p] >= 0); the
// magnitude is kept when > 0, else recomputed as make_embedding does (refined_vector over the
// first dim bits, same IEEE double operation order as fill_synthetic_kernel); a magnitude that
// is still not > 0 is counted in bad[0] (IndexBuilder: keyword has zero magnitude), a
// non-finite one in bad[1] (documented deviation: the store requires finite magnitudes).
__global__ void rbee_scatter_kernel(const uint32_t* __restrict__ rec, uint64_t rec0, uint64_t n, uint32_t P,
                                    const int32_t* __restrict__ local, const PartDesc* __restrict__ parts,
                                    uint32_t dim, uint32_t kp, uint32_t wpp, uint32_t rw, PlanePerm perm,
                                    uint32_t* bad) {
    const uint32_t w32 = 2 * wpp;
    const uint64_t rec_words = 3 + uint64_t(kp) * w32;  // u32 words per record
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t g = rec0 + k;
        const int32_t li = local[g % P];
        if (li < 0) continue;
        const PartDesc& part = parts[li];
        uint32_t* planes = const_cast<uint32_t*>(part.planes);  // the store is ours to fill
        const uint64_t s = g / P;
        const uint32_t* r = rec + k * rec_words;
        const uint64_t id = uint64_t(r[0]) | (uint64_t(r[1]) << 32);
        const uint32_t* words = r + 2;
        for (uint32_t t = 0; t < kp; ++t) {
            const uint8_t* pm = perm.perm[t < uint32_t(kMaxPlanes) ? t : 0];
            uint32_t* dst = planes + (uint64_t(t) * part.count_pad + s) * w32;
            for (uint32_t h = 0; h < w32; ++h) dst[h] = permute_word(words[t * w32 + h], pm);
        }
        if (interleaved_store(int(kp), rw != 0)) {
            for (uint32_t h = 0; h < w32; ++h) {
                uint32_t w[3], z[3];
                for (uint32_t t = 0; t < 3; ++t) w[t] = planes[(uint64_t(t) * part.count_pad + s) * w32 + h];
                interleave3(w, z);
                for (uint32_t t = 0; t < 3; ++t) planes[(uint64_t(t) * part.count_pad + s) * w32 + h] = z[t];
            }
        }
        float m = __uint_as_float(r[2 + kp * w32]);
        if (!(double(m) > 0.0)) {
            double sq = 0.0;
            for (uint32_t w = 0; w < wpp; ++w) {
                const uint32_t nbits = (w + 1 == wpp && dim % 64) ? dim % 64 : 64;
                double x[64];
#pragma unroll
                for (int b = 0; b < 64; ++b) x[b] = 0.0;
                for (uint32_t t = 0; t < kp; ++t) {
                    const uint64_t v = uint64_t(words[t * w32 + 2 * w]) | (uint64_t(words[t * w32 + 2 * w + 1]) << 32);
                    const double wt = rw ? ldexp(1.0, -int(t)) : 1.0;
#pragma unroll
                    for (int b = 0; b < 64; ++b) x[b] = __dadd_rn(x[b], ((v >> b) & 1) ? wt : -wt);
                }
                for (uint32_t b = 0; b < nbits; ++b) sq = __dadd_rn(sq, __dmul_rn(x[b], x[b]));
            }
            m = __double2float_rn(__dsqrt_rn(sq));
            if (!(double(m) > 0.0)) atomicAdd(bad, 1u);
        }
        if (!isfinite(m)) atomicAdd(bad + 1, 1u);
        const_cast<float*>(part.mags)[s] = m;
        const_cast<uint64_t*>(part.ids)[s] = id;
    }
}

__global__ void count_adjacent_equal_kernel(const uint64_t* __restrict__ a, uint64_t n, uint32_t* out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i + 1 < n; i += uint64_t(gridDim.x) * blockDim.x)
        if (a[i] == a[i + 1]) atomicAdd(out, 1u);
}

__global__ void validate_mags_kernel(const float* __restrict__ mags, uint64_t count, uint32_t* bad) {
    for (uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; s < count;
         s += uint64_t(gridDim.x) * blockDim.x) {
        const float m = mags[s];
        if (!(m > 0.0f) || !isfinite(m)) atomicAdd(bad, 1u);
    }
}

// min / max of positive finite magnitudes as order-preserving u32 bit patterns
__global__ void mag_range_kernel(const float* __restrict__ mags, uint64_t count, uint32_t* out) {
    uint32_t lo = 0xffffffffu, hi = 0;
    for (uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; s < count;
         s += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t b = __float_as_uint(mags[s]);
        lo = min(lo, b);
        hi = max(hi, b);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out, lo);
        atomicMax(out + 1, hi);
    }
}

__global__ void fill_f32_kernel(float* p, uint64_t n, float v) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}

}  // namespace

void launch_repack_planes(const uint64_t* d_natural, uint32_t* d_dev, uint64_t count, uint64_t count_pad,
                          const Shape& s, const PlanePerm& perm, cudaStream_t st) {
    if (count == 0) return;
    repack_kernel<<<grid_for(count * s.w32), kThreads, 0, st>>>(d_natural, d_dev, count, count_pad, s.kp, s.wpp, s.rw,
                                                               perm);
    RBE_CK(cudaGetLastError());
}

void launch_unpack_planes(const uint32_t* d_dev, uint64_t* d_natural, uint64_t count, uint64_t count_pad,
                          const Shape& s, const PlanePerm& perm, cudaStream_t st) {
    if (count == 0) return;
    unpack_kernel<<<grid_for(count * s.wpp), kThreads, 0, st>>>(d_dev, d_natural, count, count_pad, s.kp, s.wpp, s.rw,
                                                              perm);
    RBE_CK(cudaGetLastError());
}

void launch_fill_synthetic(uint32_t* d_planes, float* d_mags, uint64_t* d_ids, uint64_t count, uint64_t count_pad,
                           uint32_t ordinal, uint32_t n_parts_total, uint64_t n_total, uint64_t seed,
                           const Shape& s, const PlanePerm& perm, cudaStream_t st) {
    if (count == 0) return;
    fill_synthetic_kernel<<<grid_for(count, 128), 128, 0, st>>>(d_planes, d_mags, d_ids, count, count_pad, ordinal,
                                                               n_parts_total, n_total, seed, s.dim, s.kp, s.wpp,
                                                               s.rw, perm);
    RBE_CK(cudaGetLastError());
}

void launch_rbee_scatter(const uint32_t* d_records, uint64_t rec0, uint64_t n, uint32_t P, const int32_t* d_local,
                         const PartDesc* d_parts, const Shape& s, const PlanePerm& perm, uint32_t* d_bad,
                         cudaStream_t st) {
    if (n == 0) return;
    rbee_scatter_kernel<<<grid_for(n, 128), 128, 0, st>>>(d_records, rec0, n, P, d_local, d_parts, s.dim, s.kp, s.wpp,
                                                         s.rw, perm, d_bad);
    RBE_CK(cudaGetLastError());
}

void launch_count_adjacent_equal(const uint64_t* d_sorted, uint64_t n, uint32_t* d_out, cudaStream_t st) {
    if (n < 2) return;
    count_adjacent_equal_kernel<<<grid_for(n), kThreads, 0, st>>>(d_sorted, n, d_out);
    RBE_CK(cudaGetLastError());
}

void launch_validate_mags(const float* d_mags, uint64_t count, uint32_t* d_bad, cudaStream_t st) {
    if (count == 0) return;
    validate_mags_kernel<<<grid_for(count), kThreads, 0, st>>>(d_mags, count, d_bad);
    RBE_CK(cudaGetLastError());
}

void launch_mag_range(const float* d_mags, uint64_t count, uint32_t* d_out, cudaStream_t st) {
    if (count == 0) return;
    mag_range_kernel<<<grid_for(count), kThreads, 0, st>>>(d_mags, count, d_out);
    RBE_CK(cudaGetLastError());
}

void launch_fill_f32(float* p, uint64_t n, float v, cudaStream_t st) {
    if (n == 0) return;
    fill_f32_kernel<<<grid_for(n), kThreads, 0, st>>>(p, n, v);
    RBE_CK(cudaGetLastError());
}

}  // namespace rbe_dev
