// tmem.cu -- B200 microbenchmark of the tensor-memory paths the tensor scan
// depends on: tcgen05.ld throughput (32x32b shapes, with and without
// .pack::16b), tcgen05.st throughput, and tcgen05.mma kind::i8 (A in TMEM,
// B in shared memory) issue rate at M=128, N=64/128/256, K=32.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/tmem tools/microbench/tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int MODE>
__global__ void __launch_bounds__(512, 1) ld_kernel(int iters, unsigned long long* cyc, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + (uint32_t((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    uint32_t acc = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t v[32];
        if (MODE == 0) {  // 64 columns as 2 x32 loads
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(base + 32 * h));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int e = 0; e < 32; ++e) acc ^= v[e];
            }
        } else {  // 64 columns as 2 x16.pack::16b loads (16 regs each, two 16-bit halves)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(base + 32 * h));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int e = 0; e < 32; ++e) acc ^= v[e];
            }
        }
    }
    const long long t1 = clock64();
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

__global__ void __launch_bounds__(512, 1) st_kernel(int iters, unsigned long long* cyc) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + (uint32_t((warp & 3) * 32) << 16) + (warp >> 2) * 64;
    uint32_t v = threadIdx.x;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int h = 0; h < 4; ++h)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                    base + 16 * h),
                "r"(v + it));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3fffu);
    d |= uint64_t(128 >> 4) << 16;
    d |= uint64_t(256 >> 4) << 32;
    d |= uint64_t(1) << 46;
    return d;
}

// one thread issues `iters` x 8 MMAs (M=128, N, K=32, kind::i8, A in TMEM) and waits at the end
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, int N, int a_tmem, int nd, unsigned long long* cyc) {
    __shared__ __align__(1024) uint8_t bsm[256 * 32];
    __shared__ __align__(1024) uint8_t asm_[128 * 32];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) bsm[i] = 1;
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) asm_[i] = 1;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t(N) >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t d_t = slot + 256, a_t = slot;
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        const uint64_t bd = smem_desc(smem_u32(bsm));
        const uint64_t ad = smem_desc(smem_u32(asm_));
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t dd = d_t + uint32_t(k % nd) * uint32_t(N);
                if (a_tmem)
                    asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;" ::"r"(dd), "r"(a_t),
                                 "l"(bd), "r"(idesc));
                else
                    asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(dd), "l"(ad),
                                 "l"(bd), "r"(idesc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n}"
                         : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
        t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

// `issuers` warps, lane 0 of each issues iters x 8 MMAs (M=128, N=64, K=32, A in TMEM) into its own D
__global__ void __launch_bounds__(128, 1) mma_multi_kernel(int iters, int issuers, unsigned long long* cyc) {
    __shared__ __align__(1024) uint8_t bsm[256 * 32];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar[4];
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) bsm[i] = 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x < 4) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[threadIdx.x])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    const long long t0 = clock64();
    if (warp < issuers && lane == 0) {
        const uint32_t d_t = slot + 256 + 64 * warp, a_t = slot + 32 * warp;
        const uint64_t bd = smem_desc(smem_u32(bsm));
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, 1;" ::"r"(d_t), "r"(a_t), "l"(bd),
                             "r"(idesc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[warp])));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n}"
                         : "=r"(ok) : "r"(smem_u32(&bar[warp])) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    unsigned long long* cyc;
    uint32_t* sink;
    CK(cudaMalloc(&cyc, 8 * 1024));
    CK(cudaMalloc(&sink, 4 * 1024 * 512));
    unsigned long long h[1024];
    const int iters = 2000;
    for (int mode = 0; mode < 2; ++mode) {
        for (int warps = 4; warps <= 16; warps *= 2) {
            if (mode == 0) ld_kernel<0><<<sms, 32 * warps>>>(iters, cyc, sink);
            else ld_kernel<1><<<sms, 32 * warps>>>(iters, cyc, sink);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost));
            double m = 0;
            for (int i = 0; i < sms; ++i) m += h[i];
            m /= sms;
            const double bytes = double(iters) * warps * 32 * 64 * 4;  // 64 columns x 32 lanes x 4 B per warp-iter
            printf("tcgen05.ld 32x32b.x32%s  warps=%2d: %.1f cycles/iter/warp, TMEM read %.1f B/clk/SM (64 cols/warp/iter)\n",
                   mode ? ".pack::16b" : "          ", warps, m / iters, bytes / m);
        }
    }
    for (int warps = 4; warps <= 16; warps *= 2) {
        st_kernel<<<sms, 32 * warps>>>(iters, cyc);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost));
        double m = 0;
        for (int i = 0; i < sms; ++i) m += h[i];
        m /= sms;
        const double bytes = double(iters) * warps * 32 * 64 * 4;
        printf("tcgen05.st 32x32b.x16 x4  warps=%2d: %.1f cycles/iter/warp, TMEM write %.1f B/clk/SM\n", warps,
               m / iters, bytes / m);
    }
    for (int a_tmem = 0; a_tmem < 2; ++a_tmem)
      for (int nd = 1; nd <= 4; nd *= 2)
        for (int N = 64; N <= 256; N *= 2) {
            if (N * nd > 256) continue;
            mma_kernel<<<sms, 128>>>(iters, N, a_tmem, nd, cyc);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost));
            double m = 0;
            for (int i = 0; i < sms; ++i) m += h[i];
            m /= sms;
            printf("tcgen05.mma kind::i8 M128 N%3d K32 A in %s, %d independent D: %.1f cycles/MMA (%.0f MAC/clk/SM)\n", N,
                   a_tmem ? "TMEM" : "SMEM", nd, m / (iters * 8.0), 128.0 * N * 32 * iters * 8 / m);
        }
    for (int issuers = 1; issuers <= 4; issuers *= 2) {
        mma_multi_kernel<<<sms, 128>>>(iters, issuers, cyc);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost));
        double m = 0;
        for (int i = 0; i < sms; ++i) m += h[i];
        m /= sms;
        printf("tcgen05.mma kind::i8 M128 N64 K32, %d issuing warps (own D each): %.1f cycles per MMA per SM\n",
               issuers, m / (iters * 8.0 * issuers));
    }
    return 0;
}
