// mma_pace.cu -- tensor-core pacing of the scan's MMA shape on B200 (M128 N64 K32 kind::i8):
// issue R rounds back to back (no waits, one commit at the end); a round is G groups of 5 MMAs
// (one group = one 128-doc sub-tile into its own accumulator D_g), issued either group by group
// ("seq": D0 k0..k4, D1 k0..k4, ...) or interleaved by K block ("ilv": D0 k0, D1 k0, ..., D0 k1, ...).
// If the ~70-cycle cost per MMA of a single chain is the accumulate dependency, interleaving
// independent accumulators should approach the 128*N/256-cycle dispatch floor.
// Also: A from shared memory (SS) instead of TMEM, and N = 128 / 256.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_pace.cu -o mma_pace
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((saddr >> 4) & 0x3fffu) | (uint64_t((lbo >> 4) & 0x3fff) << 16) |
           (uint64_t((sbo >> 4) & 0x3fff) << 32) | (uint64_t(1) << 46);
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
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
        : "memory");
}

// smem: B = N rows x 5 K blocks (N*32 B each), A (SS mode) = 128 rows x 5 K blocks (4 KB each)
__global__ void __launch_bounds__(32, 1) k(int rounds, int G, int ilv, int ss, int N, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    uint8_t* bsm = sm;
    uint8_t* asm_ = sm + 5 * 256 * 32;
    for (int i = threadIdx.x; i < (5 * 256 * 32 + 5 * 4096) / 4; i += 32) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (2u << 4) | (1u << 10) | ((uint32_t(N) >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t tb = slot;
    // TMEM: A at columns [0, 40), D_g at 64 + g * N (G * N <= 448)
    const long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
        if (ilv) {
            for (int kb = 0; kb < 5; ++kb)
                for (int g = 0; g < G; ++g) {
                    const uint32_t d = tb + 64 + g * N;
                    const uint64_t b = smem_desc(smem_u32(bsm) + kb * N * 32, 128, 256);
                    if (ss) mma_ss(d, smem_desc(smem_u32(asm_) + kb * 4096, 128, 256), b, idesc, kb > 0);
                    else mma_ts(d, tb + 8 * kb, b, idesc, kb > 0);
                }
        } else {
            for (int g = 0; g < G; ++g)
                for (int kb = 0; kb < 5; ++kb) {
                    const uint32_t d = tb + 64 + g * N;
                    const uint64_t b = smem_desc(smem_u32(bsm) + kb * N * 32, 128, 256);
                    if (ss) mma_ss(d, smem_desc(smem_u32(asm_) + kb * 4096, 128, 256), b, idesc, kb > 0);
                    else mma_ts(d, tb + 8 * kb, b, idesc, kb > 0);
                }
        }
    }
    commit(&bar);
    while (!mtry(&bar, 0)) {
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, 8 * 1024);
    unsigned long long h[1024];
    const int smem = 5 * 256 * 32 + 5 * 4096;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    struct Cfg {
        int N, G, ilv, ss;
    };
    const Cfg cfgs[] = {{64, 1, 0, 0}, {64, 2, 0, 0}, {64, 4, 0, 0}, {64, 2, 1, 0}, {64, 4, 1, 0}, {64, 6, 1, 0},
                        {64, 1, 0, 1}, {64, 4, 1, 1}, {32, 4, 1, 0}, {128, 1, 0, 0}, {128, 2, 1, 0}, {128, 3, 1, 0},
                        {256, 1, 0, 0}};
    for (const Cfg& c : cfgs) {
        const int rounds = 2000 / c.G;
        k<<<sms, 32, smem>>>(rounds, c.G, c.ilv, c.ss, c.N, d);
        if (cudaDeviceSynchronize() != cudaSuccess) {
            printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
            return 1;
        }
        cudaMemcpy(h, d, 8 * sms, cudaMemcpyDeviceToHost);
        double m = 0;
        for (int i = 0; i < sms; ++i) m += h[i];
        m /= sms;
        const double per_mma = m / (double(rounds) * c.G * 5);
        printf("N=%3d G=%d %s %s: %6.1f cycles per MMA, %6.1f per 5-MMA sub-tile (floor %d)\n", c.N, c.G,
               c.ilv ? "interleaved" : "sequential ", c.ss ? "A:smem" : "A:tmem", per_mma, per_mma * 5,
               128 * c.N / 256);
    }
    return 0;
}
