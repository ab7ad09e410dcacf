// sync.cu -- cost of the tensor scan's per-sub-tile synchronisation skeleton on B200:
// 3 warpgroups x 4 warps; per iteration each warp waits its warpgroup's "done" mbarrier,
// (optionally) waits a ring stage's "full" mbarrier fed by a producer warp and arrives on
// its "empty", then counts itself in with a shared atomic; the last of four arrives on
// "done".  Reports cycles per iteration per warpgroup.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void minit(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c)); }
__device__ __forceinline__ void marrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ bool mtry(uint64_t* b, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
    return ok;
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t par) { while (!mtry(b, par)) {} }

__global__ void __launch_bounds__(416, 1) k(int iters, int ring, int nst, unsigned long long* out) {
    __shared__ __align__(8) uint64_t done[3], full[16], empty[16];
    __shared__ uint32_t cnt[3];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int g = 0; g < 3; ++g) { minit(&done[g], 1); cnt[g] = 0; }
        for (int s = 0; s < nst; ++s) { minit(&full[s], 1); minit(&empty[s], 4); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long t0 = clock64();
    if (warp == 12) {
        if (ring && lane == 0) {
            int idx = 0, ph = 0;
            for (int i = 0; i < 3 * iters; ++i) {
                mwait(&empty[idx], ph ^ 1);
                marrive(&full[idx]);
                if (++idx == nst) { idx = 0; ph ^= 1; }
            }
        }
    } else {
        const int g = warp >> 2;
        // prime: the first "done" phase is completed by warp 0 of each group
        if ((warp & 3) == 0 && lane == 0) marrive(&done[g]);
        int u = g, sidx = u % nst, sph = (u / nst) & 1;
        for (int it = 0; it < iters; ++it) {
            mwait(&done[g], it & 1);
            if (ring) {
                mwait(&full[sidx], sph);
                __syncwarp();
                if (lane == 0) marrive(&empty[sidx]);
                sidx += 3;
                while (sidx >= nst) { sidx -= nst; sph ^= 1; }
            }
            __syncwarp();
            uint32_t old = 0;
            if (lane == 0)
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(&cnt[g])) : "memory");
            old = __shfl_sync(0xffffffffu, old, 0);
            if ((old & 3) == 3 && lane == 0) marrive(&done[g]);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, 8 * 1024);
    unsigned long long h[1024];
    for (int ring = 0; ring < 2; ++ring) {
        const int iters = 4000;
        k<<<sms, 416>>>(iters, ring, 12, d);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("err %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
        cudaMemcpy(h, d, 8 * sms, cudaMemcpyDeviceToHost);
        double m = 0;
        for (int i = 0; i < sms; ++i) m += h[i];
        m /= sms;
        printf("%s: %.0f cycles per iteration per warpgroup (3 warpgroups in parallel)\n",
               ring ? "done-barrier + atomic + ring (producer warp)" : "done-barrier + atomic only", m / iters);
    }
    return 0;
}
