// rbe_common.cuh -- definitions shared by the sm_100a kernels and the host
// orchestration of the B200 RBE retrieval path.
//
// Device store layout.  Per partition, bit-plane-major:
//   planes : u32 [keyword_planes][count_pad][W32]     W32 = 2*ceil(dim/64)
//   mags   : f32 [count_pad]                          (pad entries = 1.0f)
//   ids    : u64 [count]
// Word g of a doc plane holds dims [32g, 32g+32) of that plane, with the bits
// permuted INSIDE the word by a fixed per-plane permutation (perm[t][bit] =
// dim offset).  The permutation is chosen so the tensor-core kernel turns the
// kp plane words of a 32-dim group into the 32 per-dim bytes
// V = sum_t 2^(kp-1-t) b_t with ~25 ALU ops (see expand32 below).  All the
// reference's quantities are invariant under a common permutation of the
// positions of a doc plane and the query plane it is dotted with
// (binary_dot_words, binary_vector.hpp:33-40, sums popcounts over words).
#pragma once

#include <cstdint>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

namespace rbe_dev {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

// splitmix64 output #j of a stream seeded with `seed` (src/bench.cpp:15-21,
// counter form).
__host__ __device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t j) {
    uint64_t z = seed + (j + 1) * kGamma;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint32_t sel32(uint32_t m, uint32_t a, uint32_t b) {
    return (a & m) | (b & ~m);  // one LOP3
}

// x >> s as a multiply-high (IMAD.HI runs on the FMA pipe, leaving the
// half-rate ALU pipe to the LOP3 masks); s in [1, 31].
__host__ __device__ __forceinline__ uint32_t shr(uint32_t x, int s) {
#ifdef __CUDA_ARCH__
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(1u << (32 - s)));
    return r;
#else
    return x >> s;
#endif
}
// x << s as a multiply (IMAD on the FMA pipe)
__host__ __device__ __forceinline__ uint32_t shl(uint32_t x, int s) { return x * (1u << s); }

__host__ __device__ __forceinline__ uint32_t rotr32(uint32_t x, int r) {
    return r == 0 ? x : ((x >> r) | (x << (32 - r)));
}

// ---------------------------------------------------------------------------
// expand32<KP, RW>: kp plane words of one 32-dim group (device layout) ->
// 8 u32 words = 32 bytes, byte (4*o + k) of the output = V of dim offset
// 4*o + k.  Weighted (RW): V = sum_t 2^(kp-1-t) b_t in [0, 2^kp - 1];
// unweighted: V = sum_t b_t in [0, kp].  The device-layout permutation of each
// plane is derived on the host by probing this very function
// (derive_plane_permutation), so layout and expansion cannot disagree.
template <int KP, bool RW>
struct Expand {
    // Generic path: bit (8k + o) of every plane word -> byte (4o + k).
    __host__ __device__ __forceinline__ static void run(const uint32_t* w, uint32_t* out) {
#pragma unroll
        for (int o = 0; o < 8; ++o) {
            uint32_t v = 0;
#pragma unroll
            for (int t = 0; t < KP; ++t) {
                const uint32_t b = (o ? shr(w[t], o) : w[t]) & 0x01010101u;
                v += RW ? shl(b, KP - 1 - t) : b;
            }
            out[o] = v;
        }
    }
};

template <>
struct Expand<2, true> {
    // V = 2 b0 + b1.  Z0 takes plane 0 on odd bits, plane 1 on even bits;
    // Z1 the complement, rotated right by one.  Bit pairs (2j, 2j+1) of a byte
    // are then (b1, b0) of one dim.
    __host__ __device__ __forceinline__ static void run(const uint32_t* w, uint32_t* out) {
        const uint32_t z0 = sel32(0xAAAAAAAAu, w[0], w[1]);
        const uint32_t z1 = rotr32(sel32(0x55555555u, w[0], w[1]), 1);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            out[j] = (j ? shr(z0, 2 * j) : z0) & 0x03030303u;
            out[4 + j] = (j ? shr(z1, 2 * j) : z1) & 0x03030303u;
        }
    }
};

template <>
struct Expand<3, true> {
    // V = 4 b0 + 2 b1 + b2.  Three merged words; bit b of every byte of Z_c
    // carries plane (2 - (b - c)) mod 3, so each byte position takes each
    // plane exactly once across Z0..Z2.  Triples (plane 2,1,0) sit at bits
    // [0,3),[3,6) of Z0, [1,4),[4,7) of Z1, [2,5),[5,8) of Z2; the six
    // leftover bits form the last two dims.
    __host__ __device__ __forceinline__ static void run(const uint32_t* w, uint32_t* out) {
        const uint32_t z0 = sel32(0x24242424u, w[0], sel32(0x92929292u, w[1], w[2]));
        const uint32_t z1 = sel32(0x49494949u, w[0], sel32(0x24242424u, w[1], w[2]));
        const uint32_t z2 = sel32(0x92929292u, w[0], sel32(0x49494949u, w[1], w[2]));
        out[0] = z0 & 0x07070707u;
        out[1] = shr(z0, 3) & 0x07070707u;
        out[2] = shr(z1, 1) & 0x07070707u;
        out[3] = shr(z1, 4) & 0x07070707u;
        out[4] = shr(z2, 2) & 0x07070707u;
        out[5] = shr(z2, 5) & 0x07070707u;
        out[6] = (shr(z0, 6) & 0x03030303u) | (shl(z1, 2) & 0x04040404u);
        out[7] = (shr(z1, 7) & 0x01010101u) | (shl(z2, 1) & 0x06060606u);
    }
};

template <>
struct Expand<4, true> {
    // V = 8 b0 + 4 b1 + 2 b2 + b3, one dim per nibble.  Z_c takes plane t at
    // bit positions = c + 3 - t (mod 4); rotating right by c aligns nibbles.
    __host__ __device__ __forceinline__ static void run(const uint32_t* w, uint32_t* out) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const uint32_t m0 = 0x11111111u << ((c + 3) & 3);
            const uint32_t m1 = 0x11111111u << ((c + 2) & 3);
            const uint32_t m2 = 0x11111111u << ((c + 1) & 3);
            const uint32_t z = rotr32(sel32(m0, w[0], sel32(m1, w[1], sel32(m2, w[2], w[3]))), c);
            out[2 * c] = z & 0x0F0F0F0Fu;
            out[2 * c + 1] = shr(z, 4) & 0x0F0F0F0Fu;
        }
    }
};

// ---------------------------------------------------------------------------
// Plane interleaving (kp = 3, residual weights).  The store keeps, per 32-dim
// group, the three (permuted) plane words pre-merged as z_c, c = 0..2:
//   z0 = w0 @ 0x24.. | w1 @ 0x92.. | w2 @ 0x49..
//   z1 = w0 @ 0x49.. | w1 @ 0x24.. | w2 @ 0x92..
//   z2 = w0 @ 0x92.. | w1 @ 0x49.. | w2 @ 0x24..
// (a bijection of the same 96 bits: every bit position takes each plane once
// across z0..z2).  These are exactly the merged words Expand<3, true> builds
// first, so the tensor scan expands straight from the stored words.
__host__ __device__ __forceinline__ constexpr bool interleaved_store(int kp, bool rw) { return kp == 3 && rw; }
__host__ __device__ __forceinline__ void interleave3(const uint32_t* w, uint32_t* z) {
    z[0] = sel32(0x24242424u, w[0], sel32(0x92929292u, w[1], w[2]));
    z[1] = sel32(0x49494949u, w[0], sel32(0x24242424u, w[1], w[2]));
    z[2] = sel32(0x92929292u, w[0], sel32(0x49494949u, w[1], w[2]));
}
__host__ __device__ __forceinline__ void deinterleave3(const uint32_t* z, uint32_t* w) {
    w[0] = (z[0] & 0x24242424u) | (z[1] & 0x49494949u) | (z[2] & 0x92929292u);
    w[1] = (z[0] & 0x92929292u) | (z[1] & 0x24242424u) | (z[2] & 0x49494949u);
    w[2] = (z[0] & 0x49494949u) | (z[1] & 0x92929292u) | (z[2] & 0x24242424u);
}

// Expansion from the STORED words of a 32-dim group (interleaved for kp = 3 weighted).
template <int KP, bool RW>
struct ExpandStored {
    __host__ __device__ __forceinline__ static void run(const uint32_t* w, uint32_t* out) { Expand<KP, RW>::run(w, out); }
};
template <>
struct ExpandStored<3, true> {
    __host__ __device__ __forceinline__ static void run(const uint32_t* z, uint32_t* out) {
        out[0] = z[0] & 0x07070707u;
        out[1] = shr(z[0], 3) & 0x07070707u;
        out[2] = shr(z[1], 1) & 0x07070707u;
        out[3] = shr(z[1], 4) & 0x07070707u;
        out[4] = shr(z[2], 2) & 0x07070707u;
        out[5] = shr(z[2], 5) & 0x07070707u;
        out[6] = (shr(z[0], 6) & 0x03030303u) | (shl(z[1], 2) & 0x04040404u);
        out[7] = (shr(z[1], 7) & 0x01010101u) | (shl(z[2], 1) & 0x06060606u);
    }
};

// Runtime-dispatched host version (permutation derivation, tests).
inline void expand32_host(int kp, bool rw, const uint32_t* w, uint32_t* out) {
    if (rw) {
        switch (kp) {
            case 1: Expand<1, true>::run(w, out); return;
            case 2: Expand<2, true>::run(w, out); return;
            case 3: Expand<3, true>::run(w, out); return;
            case 4: Expand<4, true>::run(w, out); return;
            case 5: Expand<5, true>::run(w, out); return;
            case 6: Expand<6, true>::run(w, out); return;
            case 7: Expand<7, true>::run(w, out); return;
            default: Expand<8, true>::run(w, out); return;
        }
    }
    switch (kp) {
        case 1: Expand<1, false>::run(w, out); return;
        case 2: Expand<2, false>::run(w, out); return;
        case 3: Expand<3, false>::run(w, out); return;
        case 4: Expand<4, false>::run(w, out); return;
        case 5: Expand<5, false>::run(w, out); return;
        case 6: Expand<6, false>::run(w, out); return;
        case 7: Expand<7, false>::run(w, out); return;
        default: Expand<8, false>::run(w, out); return;
    }
}

// Largest keyword plane count with a tensor-core expansion (V fits u8).
constexpr int kMaxTensorPlanes = 8;
// Permutations are defined for every kp; above 8 planes (no tensor path) the
// identity is used.
constexpr int kMaxPlanes = 64;

// ---------------------------------------------------------------------------
// Device-side partition descriptor.
struct PartDesc {
    const uint32_t* planes;  // [kp][count_pad][W32]
    const float* mags;       // [count_pad]
    const uint64_t* ids;     // [count]
    uint64_t count;
    uint64_t count_pad;
    uint32_t ordinal;
    uint32_t pad_;
};

// Survivor / result record (== rbe_result in include/rbe_cuda.h).
struct Result {
    double score;
    uint64_t id;
    int64_t acc;
    uint32_t partition;
    uint32_t valid;
};

// Order key of (score desc, id asc) (entry_less, search.cpp:50-53) as two
// u64 compared lexicographically ascending.  -0.0 is folded into +0.0 so the
// key order equals the reference's double comparison.
__host__ __device__ __forceinline__ uint64_t score_desc_key(double s) {
    if (s == 0.0) s = 0.0;
    uint64_t b;
#ifdef __CUDA_ARCH__
    b = (uint64_t)__double_as_longlong(s);
#else
    __builtin_memcpy(&b, &s, 8);
#endif
    const uint64_t asc = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    return ~asc;
}

}  // namespace rbe_dev
