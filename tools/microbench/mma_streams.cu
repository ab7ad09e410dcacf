// mma_streams.cu -- tensor-core throughput for the scan's MMA shape (kind::i8, M128, K32, A in
// TMEM, B in smem) as a function of the number of issuing warps W and N: each warp streams
// groups of 5 accumulating MMAs into its own pair of accumulators (commit per group, waits only
// before reusing an accumulator).  Prints cycles per MMA per SM.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_streams.cu -o mma_streams
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ bool mtry(uint64_t* b, uint32_t par) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(par)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3fffu) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) |
           (uint64_t(1) << 46);
}

template <int W, int N>
__global__ void __launch_bounds__(32 * W, 1) k(int groups, unsigned long long* out) {
    static_assert(40 + N * 2 * W <= 512, "TMEM");
    __shared__ __align__(1024) uint8_t bsm[5 * 256 * 32];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bars[2 * W];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 5 * 256 * 32 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(bsm)[i] = 0x01010101u;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2 * W; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // TMEM: A at columns [0, 40) (shared by all), D pairs after: warp w uses D at 40 + N * (2w + s)
    constexpr uint32_t idesc = (2u << 4) | (1u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t b0 = sdesc(su32(bsm));
    uint32_t ph[2] = {0, 0};
    const long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
        const int s = g & 1;
        if (g >= 2) {
            while (!mtry(&bars[2 * warp + s], ph[s])) {
            }
            ph[s] ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        const uint32_t dt = 40 + N * (2 * warp + s);
#pragma unroll
        for (int kb = 0; kb < 5; ++kb)
            asm volatile(
                "{\n\t.reg .pred q, e;\n\tsetp.ne.b32 q, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, q;\n}" ::"r"(dt),
                "r"(8 * kb), "l"(b0 + kb * ((N * 32) >> 4)), "r"(idesc), "r"(kb)
                : "memory");
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
                su32(&bars[2 * warp + s]))
            : "memory");
    }
    for (int s = 0; s < 2; ++s)
        while (!mtry(&bars[2 * warp + s], ph[s])) {
        }
    const long long t1 = clock64();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
    }
}

template <int W, int N>
void run(unsigned long long* d, int sms) {
    const int groups = 2000;
    k<W, N><<<sms, 32 * W>>>(groups, d);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
        return;
    }
    unsigned long long h[256];
    cudaMemcpy(h, d, 8 * sms, cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < sms; ++i) c += h[i];
    c /= sms;
    printf("W=%d N=%3d: %6.1f cycles per MMA per SM (%.0f MAC/clk/SM)\n", W, N, c / (groups * 5.0 * W),
           128.0 * N * 32 * groups * 5.0 * W / c);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, 8 * 256);
    run<1, 64>(d, sms);
    run<2, 64>(d, sms);
    run<3, 64>(d, sms);
    run<1, 128>(d, sms);
    run<1, 32>(d, sms);
    run<2, 32>(d, sms);
    run<4, 32>(d, sms);
    return 0;
}
