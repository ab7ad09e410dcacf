// mma_contend.cu -- does TMEM load/store traffic from the CUDA cores slow the tensor core?
// One issuer warp streams the scan's MMA groups (5 x M128 N64 K32 kind::i8, A in TMEM, 4
// accumulators used round robin, at most 4 groups in flight) while 16 worker warps hammer
// TMEM: mode 0 idle, 1 tcgen05.ld x32.pack::16b of 64 columns (the scan's test epilogue),
// 2 tcgen05.st x16 x2 = 32 columns (the scan's expand), 3 both.  Reports cycles per MMA group
// and the workers' TMEM bytes per cycle per SM.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_contend.cu -o mma_contend
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3fffu) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (uint64_t(1) << 46);
}
__device__ __forceinline__ bool mtry(uint64_t* b, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n}"
                 : "=r"(ok)
                 : "r"(smem_u32(b)), "r"(par)
                 : "memory");
    return ok;
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(544, 1) k(int groups, int mode, int nworkers, unsigned long long* out) {
    __shared__ __align__(1024) uint8_t bsm[5 * 64 * 32];
    __shared__ uint32_t slot;
    __shared__ volatile uint32_t stop;
    __shared__ __align__(8) uint64_t bars[4];
    __shared__ unsigned long long wops;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 5 * 64 * 32 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bsm)[i] = 0x01010101u;
    if (threadIdx.x == 0) {
        stop = 0;
        wops = 0;
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 16) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = slot;
    if (warp == 16) {
        const uint32_t idesc = (2u << 4) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
        uint32_t ph[4] = {0, 0, 0, 0};
        const long long t0 = clock64();
        for (int g = 0; g < groups; ++g) {
            const int s = g & 3;
            if (g >= 4) {
                while (!mtry(&bars[s], ph[s])) {
                }
                ph[s] ^= 1;
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            for (int kb = 0; kb < 5; ++kb)
                mma_ts(tb + 64 + 64 * s, tb + 8 * kb, smem_desc(smem_u32(bsm) + kb * 64 * 32), idesc, kb > 0);
            commit(&bars[s]);
        }
        for (int s = 0; s < 4; ++s) {
            while (!mtry(&bars[s], ph[s])) {
            }
        }
        const long long t1 = clock64();
        stop = 1;
        if (lane == 0) out[blockIdx.x * 2] = t1 - t0;
    } else if (warp < nworkers) {
        const uint32_t lane_base = uint32_t((warp & 3) * 32) << 16;
        const uint32_t ldc = tb + lane_base + 320;  // 64 columns read
        const uint32_t stc = tb + lane_base + 384 + 32 * ((warp >> 2) & 3) / 2;  // 32 columns written
        unsigned long long ops = 0;
        uint32_t sink = 0;
        uint32_t v[32];
        for (int i = 0; i < 32; ++i) v[i] = i * lane;
        while (!stop) {
            if (mode & 1) {
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                    "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                      "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                      "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                      "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                      "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                    : "r"(ldc)
                    : "memory");
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                sink ^= v[0] & v[31];
            }
            if (mode & 2) {
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16};" ::"r"(stc),
                    "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                    "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                    : "memory");
                asm volatile(
                    "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16};" ::"r"(stc + 16),
                    "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
                    "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
                    : "memory");
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            if (mode == 0) break;
            ++ops;
        }
        if (lane == 0) atomicAdd(&wops, ops);
        if (sink == 0x12345) out[1] = sink;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x * 2 + 1] = wops;
    if (warp == 16) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
    }
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, 16 * 1024);
    unsigned long long h[2048];
    const char* names[] = {"idle", "ld64 pack16", "st32", "ld64+st32"};
    for (int nw : {4, 16})
        for (int mode = 0; mode < 4; ++mode) {
            if (nw == 4 && mode == 0) continue;
            const int groups = 4000;
            k<<<sms, 544>>>(groups, mode, nw, d);
            if (cudaDeviceSynchronize() != cudaSuccess) {
                printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
                return 1;
            }
            cudaMemcpy(h, d, 16 * sms, cudaMemcpyDeviceToHost);
            double cyc = 0, ops = 0;
            for (int i = 0; i < sms; ++i) {
                cyc += h[2 * i];
                ops += h[2 * i + 1];
            }
            cyc /= sms;
            ops /= sms;
            const double bytes_per_op = ((mode & 1) ? 64 * 32 * 4 : 0) + ((mode & 2) ? 32 * 32 * 4 : 0);
            printf("workers=%2d %-12s: %6.1f cycles per 5-MMA group; worker TMEM traffic %6.1f B/clk/SM "
                   "(%.1f worker ops per group)\n",
                   nw, names[mode], cyc / groups, ops * bytes_per_op / cyc, ops / groups);
        }
    return 0;
}
