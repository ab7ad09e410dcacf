// pipe_v3.cu -- warp-specialised scan pipeline prototype, unit = one 256-doc ring stage
// (two 128-doc sub-tiles): producer warp (two cp.async.bulk per stage from a doc-major store:
// planes [count][3][4] u32, mags [count] f32), NI MMA-issuer warps (10 MMAs per stage), NE
// expander warpgroups (two docs per thread), NT tester warpgroups (one 128-column tcgen05.ld per
// stage).  NAS A-stage buffers (2 x 40 TMEM columns) and NDS D-stage buffers (2 x 64 columns).
// Prints ms, GB/s of the 52 B/doc stream and cycles per 256-doc stage per SM.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1802_06466_b200/csrc pipe_v3.cu -o pipe_v3
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <type_traits>
#include <cuda_runtime.h>

#include "rbe_common.cuh"

using namespace rbe_dev;

constexpr int NS = 12;
constexpr int STAGE_BYTES = 3 * 4096 + 1024;

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void marrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mexpect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mtry(uint64_t* b, uint32_t par) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(par)
        : "memory");
    return ok != 0;
}
// wait with a hardware suspend hint (the warp sleeps until the phase completes instead of
// spinning); traps after ~minutes so a protocol bug cannot hang the GPU
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t par) {
    uint32_t n = 0, ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(su32(b)), "r"(par), "r"(1000000u)
            : "memory");
        if (++n == (1u << 20)) {
            printf("stuck block %d warp %d bar %u par %u\n", blockIdx.x, threadIdx.x >> 5, su32(b), par);
            asm volatile("trap;");
        }
    } while (!ok);
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void fb() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fa() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void st16(uint32_t t, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16};" ::"r"(t),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void st2(uint32_t t, uint32_t a, uint32_t b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(t), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void st8(uint32_t t, uint32_t a) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(t), "r"(a)
                 : "memory");
}
#define R8(o) "=r"(v[o]), "=r"(v[o + 1]), "=r"(v[o + 2]), "=r"(v[o + 3]), "=r"(v[o + 4]), "=r"(v[o + 5]), "=r"(v[o + 6]), "=r"(v[o + 7])
__device__ __forceinline__ void ld64p(uint32_t t, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.pack::16b.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, "
        "%36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, "
        "%58, %59, %60, %61, %62, %63}, [%64];"
        : R8(0), R8(8), R8(16), R8(24), R8(32), R8(40), R8(48), R8(56)
        : "r"(t)
        : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3fffu) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
           (uint64_t(1) << 46);
}
// ring position (index, parity) advanced by a fixed step
template <int N>
struct Pos {
    uint32_t i = 0, ph = 0;
    __device__ __forceinline__ void adv(uint32_t step) {
        i += step;
        while (i >= uint32_t(N)) {
            i -= N;
            ph ^= 1;
        }
    }
};

struct P {
    const uint32_t* planes;  // [count][3][4]
    const float* mags;
    uint32_t ntiles;
    int mode;  // bit0: no MMA, bit1: no expand math
    unsigned long long* out;
    unsigned long long* prof;  // [grid][32 warps][4]
};

template <int NE, int NT, int NI, int NAS, int NDS>
__global__ void __launch_bounds__(32 * (4 + 4 * (NE + NT)), 1) pipe(P p) {
    static_assert(NAS * 80 + NDS * 128 <= 512, "TMEM");
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* ring = sm;
    uint8_t* bsm = sm + NS * STAGE_BYTES;  // 5 K blocks of B (64 x 32 B), 10 KB
    uint64_t* full = reinterpret_cast<uint64_t*>(bsm + 5 * 2048);
    uint64_t* empty = full + NS;
    uint64_t* afull = empty + NS;
    uint64_t* aempty = afull + NAS;
    uint64_t* dfull = aempty + NAS;
    uint64_t* dempty = dfull + NDS;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(dempty + NDS);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 5 * 2048 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(bsm)[i] = i >= 4 * 512 ? 1u : 0x01ff02feu * (i | 1);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            minit(full + s, 1);
            minit(empty + s, 4);
        }
        for (int a = 0; a < NAS; ++a) {
            minit(afull + a, 4);
            minit(aempty + a, 2);
        }
        for (int d = 0; d < NDS; ++d) {
            minit(dfull + d, 2);
            minit(dempty + d, 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fb();
    __syncthreads();
    fa();
    const uint32_t tb = *tslot;
    if (tb != 0) asm volatile("trap;");
    const uint32_t dbase = tb + NAS * 80;
    const uint32_t t0 = uint64_t(p.ntiles) * blockIdx.x / gridDim.x, t1 = uint64_t(p.ntiles) * (blockIdx.x + 1) / gridDim.x;
    const uint32_t nst = t1 - t0;
    const long long c0 = clock64();
    unsigned long long sink = 0;
    long long pa[4] = {0, 0, 0, 0};
#define T(slot, ...) { const long long t_ = clock64(); __VA_ARGS__; pa[slot] += clock64() - t_; }
    if (warp == 0) {
        if (lane == 0) {
            Pos<NS> r;
            for (uint32_t i = 0; i < nst; ++i, r.adv(1)) {
                if (i >= uint32_t(NS)) T(0, mwait(empty + r.i, r.ph ^ 1));
                mexpect(full + r.i, STAGE_BYTES);
                uint8_t* dst = ring + r.i * STAGE_BYTES;
                bulk(dst, p.planes + uint64_t(t0 + i) * 256 * 12, 3 * 4096, full + r.i);
                bulk(dst + 3 * 4096, p.mags + uint64_t(t0 + i) * 256, 1024, full + r.i);
            }
        }
    } else if (warp >= 1 && warp <= 2) {
        // issuer h issues the 5 MMAs of sub-tile h of every stage (two issue streams per stage)
        auto issue = [&](auto H) {
            constexpr uint32_t h = decltype(H)::value;
            const uint32_t idesc = (2u << 4) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
            const uint64_t b0 = sdesc(su32(bsm));
            Pos<NAS> a;
            Pos<NDS> d;
            for (uint32_t i = 0; i < nst; ++i, a.adv(1), d.adv(1)) {
                T(0, mwait(afull + a.i, a.ph));
                if (i >= uint32_t(NDS)) T(1, mwait(dempty + d.i, d.ph ^ 1));
                const long long ti_ = clock64();
                fa();
                if (!(p.mode & 1)) {
                    const uint32_t at = a.i * 80 + h * 40, dt = NAS * 80 + d.i * 128 + h * 64;
#pragma unroll
                    for (int kb = 0; kb < 5; ++kb)
                        asm volatile(
                            "{\n\t.reg .pred q, e;\n\tsetp.ne.b32 q, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                            "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, q;\n}" ::"r"(dt),
                            "r"(at + 8 * kb), "l"(b0 + kb * (2048 >> 4)), "r"(idesc), "r"(kb)
                            : "memory");
                }
                asm volatile(
                    "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t"
                    "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%1];\n}" ::"r"(
                        su32(aempty + a.i)),
                    "r"(su32(dfull + d.i))
                    : "memory");
                pa[2] += clock64() - ti_;
            }
        };
        if (warp == 1) issue(std::integral_constant<uint32_t, 0>{});
        else issue(std::integral_constant<uint32_t, 1>{});
    } else if (warp >= 4 && warp < 4 + 4 * NE) {
        const uint32_t eg = (warp - 4) >> 2, q = warp & 3;
        const uint32_t lb = uint32_t(q * 32) << 16;
        if (eg == 0)
            for (int a = 0; a < NAS; ++a) {
                st8(tb + lb + a * 80 + 32, ~0u);
                st8(tb + lb + a * 80 + 72, ~0u);
            }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        Pos<NS> r;
        Pos<NAS> a;
        r.adv(eg);
        a.adv(eg);
        for (uint32_t i = eg; i < nst; i += NE, r.adv(NE), a.adv(NE)) {
            T(0, mwait(full + r.i, r.ph));
            const long long te_ = clock64();
            const uint8_t* stg = ring + r.i * STAGE_BYTES;
            uint32_t out[2][32], xw[2][2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t col = h * 128 + q * 32 + lane;
                const uint4* s3 = reinterpret_cast<const uint4*>(stg) + col * 3;
                const uint4 v0 = s3[0], v1 = s3[1], v2 = s3[2];
                const float m = reinterpret_cast<const float*>(stg + 3 * 4096)[col];
                if (p.mode & 8) {
                    const uint32_t z0[4] = {v0.x, v0.y, v0.z, v0.w}, z1[4] = {v1.x, v1.y, v1.z, v1.w}, z2[4] = {v2.x, v2.y, v2.z, v2.w};
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        uint32_t* o = out[h] + 8 * g;
                        o[0] = z0[g] & 0x07070707u;
                        o[1] = (z0[g] >> 3) & 0x07070707u;
                        o[2] = (z1[g] >> 1) & 0x07070707u;
                        o[3] = (z1[g] >> 4) & 0x07070707u;
                        o[4] = (z2[g] >> 2) & 0x07070707u;
                        o[5] = (z2[g] >> 5) & 0x07070707u;
                        o[6] = ((z0[g] >> 6) & 0x03030303u) | ((z1[g] << 2) & 0x04040404u);
                        o[7] = ((z1[g] >> 7) & 0x01010101u) | ((z2[g] << 1) & 0x06060606u);
                    }
                } else if (!(p.mode & 2)) {
                    uint32_t w[3];
                    w[0] = v0.x; w[1] = v1.x; w[2] = v2.x;
                    ExpandStored<3, true>::run(w, out[h]);
                    w[0] = v0.y; w[1] = v1.y; w[2] = v2.y;
                    ExpandStored<3, true>::run(w, out[h] + 8);
                    w[0] = v0.z; w[1] = v1.z; w[2] = v2.z;
                    ExpandStored<3, true>::run(w, out[h] + 16);
                    w[0] = v0.w; w[1] = v1.w; w[2] = v2.w;
                    ExpandStored<3, true>::run(w, out[h] + 24);
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) out[h][e] = v0.x ^ v1.y ^ v2.z ^ e;
                }
                float vb = __fmaf_rz(m - 0.5f, 170.0f, -1.0e-3f);
                vb = fminf(fmaxf(vb, 0.0f), 255.0f);
                const uint32_t j = uint32_t(__float2int_rz(vb));
                xw[h][0] = j * 0x01010101u;
                xw[h][1] = (j >> 4) | 0x100u;
            }
            __syncwarp();
            if (lane == 0) marrive(empty + r.i);
            pa[1] += clock64() - te_;
            if (i >= uint32_t(NAS)) T(2, mwait(aempty + a.i, a.ph ^ 1));
            const long long ts_ = clock64();
            fa();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t at = tb + lb + a.i * 80 + h * 40;
                st16(at, out[h]);
                st16(at + 16, out[h] + 16);
                st2(at + 32, xw[h][0], xw[h][1]);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            fb();
            __syncwarp();
            if (lane == 0) marrive(afull + a.i);
            pa[3] += clock64() - ts_;
        }
    } else if (warp >= 4 + 4 * NE) {
        const uint32_t tg = (warp - 4 - 4 * NE) >> 2, q = warp & 3;
        const uint32_t lb = uint32_t(q * 32) << 16;
        Pos<NDS> d;
        d.adv(tg);
        for (uint32_t i = tg; i < nst; i += NT, d.adv(NT)) {
            T(0, mwait(dfull + d.i, d.ph));
            fa();
            uint32_t R[64];
            T(1, ld64p(dbase + lb + d.i * 128, R); asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"));
            fb();
            __syncwarp();
            if (lane == 0) marrive(dempty + d.i);
            uint32_t all = R[0], all2 = R[32];
#pragma unroll
            for (int e = 1; e < 32; ++e) {
                all &= R[e];
                all2 &= R[32 + e];
            }
            const uint32_t g = uint32_t((~all & 0x80008000u) != 0) | (uint32_t((~all2 & 0x80008000u) != 0) << 1);
            if (__any_sync(0xffffffffu, g != 0)) sink += 1;
        }
    }
    fb();
    __syncthreads();
    const long long c1 = clock64();
    if (threadIdx.x == 0) {
        p.out[blockIdx.x * 2] = c1 - c0;
        p.out[blockIdx.x * 2 + 1] = nst;
    }
    if (sink == 0xdeadbeef) p.out[0] = sink;
    if (lane == 0)
        for (int k2 = 0; k2 < 4; ++k2) p.prof[(blockIdx.x * 32 + warp) * 4 + k2] = pa[k2];
    if (warp == 0) {
        fa();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
    }
}

int main(int argc, char** argv) {
    setvbuf(stdout, NULL, _IOLBF, 0);
    const uint64_t count = argc > 1 ? strtoull(argv[1], 0, 10) : 100000000ull;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* planes;
    float* mags;
    cudaMalloc(&planes, count * 48);
    cudaMalloc(&mags, count * 4);
    cudaMemset(planes, 0x5a, count * 48);
    std::vector<float> hm(1 << 20);
    for (size_t i = 0; i < hm.size(); ++i) hm[i] = 0.5f + (i % 997) * 1e-3f;
    for (uint64_t o = 0; o < count; o += hm.size())
        cudaMemcpy(mags + o, hm.data(), std::min<uint64_t>(hm.size(), count - o) * 4, cudaMemcpyHostToDevice);
    unsigned long long* out;
    cudaMalloc(&out, sms * 16);
    unsigned long long* prof;
    cudaMalloc(&prof, sms * 32 * 4 * 8);
    std::vector<unsigned long long> hp(sms * 32 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<unsigned long long> h(sms * 2);
    const size_t smem = NS * STAGE_BYTES + 5 * 2048 + 1024;
    auto run = [&](auto kern, const char* name, int threads, int mode) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        cudaMemset(prof, 0, sms * 32 * 32);
        P p{planes, mags, uint32_t(count / 256), mode, out, prof};
        kern<<<sms, threads, smem>>>(p);
        cudaEventRecord(e0);
        kern<<<sms, threads, smem>>>(p);
        cudaEventRecord(e1);
        if (cudaEventSynchronize(e1) != cudaSuccess) {
            printf("%s err %s\n", name, cudaGetErrorString(cudaGetLastError()));
            exit(1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaMemcpy(h.data(), out, sms * 16, cudaMemcpyDeviceToHost);
        double cyc = 0, st = 0;
        for (int i = 0; i < sms; ++i) {
            cyc = std::max(cyc, double(h[2 * i]));
            st += h[2 * i + 1];
        }
        printf("%-22s mode=%d: %.3f ms  %.0f GB/s  %.1f cycles per stage per SM\n", name, mode, ms,
               count * 52.0 / ms / 1e6, cyc / (st / sms));
        cudaMemcpy(hp.data(), prof, hp.size() * 8, cudaMemcpyDeviceToHost);
        for (int w = 0; w < threads / 32; ++w) {
            double v[4] = {0, 0, 0, 0};
            for (int b = 0; b < sms; ++b)
                for (int k2 = 0; k2 < 4; ++k2) v[k2] += hp[(b * 32 + w) * 4 + k2];
            if (v[0] + v[1] + v[2] + v[3] == 0) continue;
            printf("   warp %2d per stage:", w);
            for (int k2 = 0; k2 < 4; ++k2) printf(" %7.1f", v[k2] / st);
            printf("\n");
        }
    };
#define RUN(NE, NT, NI, NAS, NDS)                                                                        \
    for (int mode : {8})                                                                        \
        run(pipe<NE, NT, NI, NAS, NDS>, "NE" #NE " NT" #NT " NI" #NI " NAS" #NAS " NDS" #NDS, 32 * (4 + 4 * (NE + NT)), mode);
    RUN(2, 1, 2, 2, 2)
    return 0;
}
