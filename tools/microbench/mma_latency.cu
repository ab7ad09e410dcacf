// mma_latency.cu -- round-trip latency of one tensor-scan MMA group on B200:
// issue 5 x tcgen05.mma kind::i8 (M128 N64 K32, A in TMEM) + commit, then wait on the
// mbarrier; with 1..4 groups in flight (independent D) to show how much overlap helps.
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
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ void group(uint32_t d, uint32_t a, uint64_t b0, uint64_t step, uint32_t idesc, uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e, p0, p1;\n\t.reg .b64 b1, b2, b3, b4;\n\t.reg .b32 a1, a2, a3, a4;\n\t"
        "setp.ne.b32 p0, 0, 0;\n\tsetp.eq.b32 p1, 0, 0;\n\t"
        "add.s64 b1, %2, %3;\n\tadd.s64 b2, b1, %3;\n\tadd.s64 b3, b2, %3;\n\tadd.s64 b4, b3, %3;\n\t"
        "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\tadd.u32 a4, %1, 32;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, p0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, p1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a2], b2, %4, p1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a3], b3, %4, p1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a4], b4, %4, p1;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n}" ::"r"(d),
        "r"(a), "l"(b0), "l"(step), "r"(idesc), "r"(smem_u32(bar))
        : "memory");
}

__global__ void __launch_bounds__(32, 1) k(int iters, int inflight, unsigned long long* out, int N) {
    __shared__ __align__(1024) uint8_t bsm[5 * 256 * 32];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bars[8];
    for (int i = threadIdx.x; i < 5 * 256 * 32; i += 32) bsm[i] = 1;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    if (threadIdx.x < 8) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[threadIdx.x])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (2u << 4) | (1u << 10) | ((uint32_t(N) >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t b0 = smem_desc(smem_u32(bsm)), step = (N * 32) >> 4;
    const long long t0 = clock64();
    uint32_t ph[4] = {0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
        const int s = it % inflight;
        if (it >= inflight) {  // wait for the group issued `inflight` groups ago on this slot
            while (!mtry(&bars[s], ph[s])) {
            }
            ph[s] ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        group(slot + 160 + (N == 64 ? 64 * s : 0), slot + 40 * s, b0, step, idesc, &bars[s]);
    }
    for (int s = 0; s < inflight && s < iters; ++s) {
        while (!mtry(&bars[s], ph[s])) {
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, 8 * 1024);
    unsigned long long h[1024];
    for (int N : {64, 128, 256})
    for (int inflight = 1; inflight <= (N == 64 ? 4 : 1); ++inflight) {
        const int iters = 2000;
        k<<<sms, 32>>>(iters, inflight, d, N);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("err %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
        cudaMemcpy(h, d, 8 * sms, cudaMemcpyDeviceToHost);
        double m = 0;
        for (int i = 0; i < sms; ++i) m += h[i];
        m /= sms;
        printf("N=%d groups in flight %d: %.0f cycles per 5-MMA group (M128 K32 i8, A in TMEM)\n", N, inflight, m / iters);
    }
    return 0;
}
