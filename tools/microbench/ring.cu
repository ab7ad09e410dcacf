// ring.cu -- B200 microbenchmark of the tensor scan's data supply alone: one
// producer thread per SM streams the bit-plane-major store (3 planes x 16 B
// per doc + f32 magnitudes, 100M docs) into a shared-memory ring with
// cp.async.bulk, one consumer warp releases the slots.  Measures the HBM
// bandwidth this access pattern reaches for different stage sizes.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/ring tools/microbench/ring.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) { while (!mbar_try(b, par)) {} }

constexpr int kDocs = 100000000;
constexpr int kStagesMax = 32;

// docs_per_stage in {128, 256, 512, 1024}; half_tiles: 1 = the current strip mapping (128 of every 256 docs)
__global__ void __launch_bounds__(64, 1) ring_kernel(const uint4* planes, const float* mags, int count_pad,
                                                     int docs_per_stage, int nst, int half_tiles,
                                                     unsigned long long* out) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t full[kStagesMax], empty[kStagesMax];
    const int stage_bytes = docs_per_stage * (3 * 16 + 4);
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // work units: contiguous runs of docs_per_stage docs; with half_tiles, unit k covers
    // docs [256*(k/ (dps/128)) ...] -- emulated as stride-2 half tiles of 128 docs
    const long long units = half_tiles ? (kDocs / 128) : (kDocs / docs_per_stage);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long sink = 0;
    const long long per_cta = (units + gridDim.x - 1) / gridDim.x;
    const long long u_begin = blockIdx.x * per_cta, u_end = min(units, u_begin + per_cta);
    if (warp == 0) {
        if (lane == 0) {
            int idx = 0, ph = 0;
            for (long long u = u_begin; u < u_end; ++u) {
                mbar_wait(empty + idx, ph ^ 1);
                long long d0;
                int nd;
                if (half_tiles) {  // strip h = u % 2 of tile ... : doc = 256*(u/2 within block) + 128*h
                    const long long blk = u / 1024, rem = u % 1024;  // 512 tiles x 2 halves per block of 131072?
                    const long long h = rem / 512, i = rem % 512;
                    d0 = blk * 131072 + i * 256 + 128 * h;
                    nd = 128;
                } else {
                    d0 = u * docs_per_stage;
                    nd = docs_per_stage;
                }
                const uint32_t bytes = nd * 52;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + idx)),
                             "r"(bytes) : "memory");
                uint8_t* dst = sm + idx * stage_bytes;
                for (int t = 0; t < 3; ++t)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(dst + t * nd * 16)),
                        "l"(planes + (long long)t * count_pad + d0), "r"(nd * 16), "r"(smem_u32(full + idx))
                        : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                                 "r"(smem_u32(dst + 3 * nd * 16)),
                             "l"(mags + d0), "r"(nd * 4), "r"(smem_u32(full + idx))
                             : "memory");
                if (++idx == nst) { idx = 0; ph ^= 1; }
            }
        }
    } else {
        int idx = 0, ph = 0;
        for (long long u = u_begin; u < u_end; ++u) {
            mbar_wait(full + idx, ph);
            sink += reinterpret_cast<const uint32_t*>(sm + idx * stage_bytes)[lane];
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + idx)) : "memory");
            if (++idx == nst) { idx = 0; ph ^= 1; }
        }
        if (lane == 0) out[blockIdx.x] = sink;
    }
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const long long count_pad = kDocs + 4096;
    uint4* planes;
    float* mags;
    unsigned long long* out;
    CK(cudaMalloc(&planes, 3 * count_pad * 16));
    CK(cudaMalloc(&mags, count_pad * 4));
    CK(cudaMalloc(&out, 8 * 1024));
    CK(cudaMemset(planes, 1, 3 * count_pad * 16));
    CK(cudaMemset(mags, 0, count_pad * 4));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct Cfg { int dps, nst, half; } cfgs[] = {{128, 12, 1}, {128, 24, 1}, {128, 12, 0}, {256, 8, 0}, {256, 16, 0},
                                                 {512, 4, 0},  {512, 8, 0},  {1024, 4, 0}};
    for (auto c : cfgs) {
        const int smem = c.nst * c.dps * 52;
        CK(cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            ring_kernel<<<sms, 64, smem>>>(planes, mags, int(count_pad), c.dps, c.nst, c.half, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("docs/stage %4d stages %2d %s: %.3f ms  %.0f GB/s\n", c.dps, c.nst, c.half ? "half-tile strips" : "contiguous      ",
               best, kDocs * 52.0 / best / 1e6);
    }
    return 0;
}
