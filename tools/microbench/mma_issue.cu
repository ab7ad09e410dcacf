// mma_issue.cu -- cost of issuing the tensor scan's per-sub-tile MMA group from one
// thread: 5 x tcgen05.mma kind::i8 (M128 N64 K32, A in TMEM, 5 distinct B K-blocks)
// with variants: + commit(s), + tcgen05.fence::after_thread_sync, + mbarrier waits.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    return uint64_t((saddr >> 4) & 0x3fffu) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (uint64_t(1) << 46);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
// whole warp executes; one elected lane issues (operands warp-uniform)
__device__ __forceinline__ void mma_i8_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mtry(uint64_t* b, uint32_t par) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
    return ok;
}

__global__ void __launch_bounds__(128, 1) k(int iters, int variant, int nkb, unsigned long long* cyc) {
    __shared__ __align__(1024) uint8_t bsm[5 * 64 * 32];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bars[8];
    for (int i = threadIdx.x; i < 5 * 64 * 32; i += blockDim.x) bsm[i] = 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x < 8) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[threadIdx.x])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (2u << 4) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    if (warp == 0 && variant >= 5) {
        // the whole warp runs the loop (operands stay warp-uniform), one elected lane issues
        const uint64_t b0 = smem_desc(smem_u32(bsm)), bstep = (64 * 32) >> 4;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t s = it & 3;
            const uint32_t a = slot + s * 40, d = slot + 160 + s * 64;
            if (it >= 4 && variant == 5) {
                while (!mtry(&bars[s], ((it >> 2) - 1) & 1)) {
                }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            uint64_t bd = b0;
            if (variant == 7) {  // compile-time 5, unrolled
#pragma unroll
                for (int kb = 0; kb < 5; ++kb, bd += bstep) mma_i8_elect(d, a + 8 * kb, bd, idesc, kb > 0);
            } else {
                for (int kb = 0; kb < nkb; ++kb, bd += bstep) mma_i8_elect(d, a + 8 * kb, bd, idesc, kb > 0);
            }
            if (variant == 5) {
                commit_elect(&bars[s]);
                commit_elect(&bars[4 + s]);
            }
        }
        if (lane == 0) {
            commit(&bars[7]);
            while (!mtry(&bars[7], 0)) {
            }
            cyc[blockIdx.x] = clock64() - t0;
        }
    } else if (threadIdx.x == 0 && variant != 5) {
        const uint64_t b0 = smem_desc(smem_u32(bsm)), bstep = (64 * 32) >> 4;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint32_t s = it & 3;
            const uint32_t a = slot + s * 40, d = slot + 160 + s * 64;
            if (variant >= 3 && variant < 6 && it >= 4) {  // wait for the group that used this slot 4 iterations ago
                while (!mtry(&bars[s], ((it >> 2) - 1) & 1)) {
                }
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            } else if (variant >= 2 && variant < 6) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            uint64_t bd = b0;
            if (variant == 6)
                for (int kb = 0; kb < nkb; ++kb) mma_i8(d, a + 8 * kb, b0, idesc, kb > 0);
            else if (variant == 7)
                for (int kb = 0; kb < nkb; ++kb, bd += bstep) mma_i8(d, a, bd, idesc, kb > 0);
            else if (variant == 8)
                for (int kb = 0; kb < nkb; ++kb, bd += bstep) mma_i8(d, a + 8 * kb, bd, idesc, 1);
            else if (variant == 9)
                for (int kb = 0; kb < nkb; ++kb) mma_i8(d, a, b0, idesc, 1);
            else
                for (int kb = 0; kb < nkb; ++kb, bd += bstep) mma_i8(d, a + 8 * kb, bd, idesc, kb > 0);
            if (variant >= 1 && variant < 6) {
                commit(&bars[s]);
                if (variant >= 4) commit(&bars[4 + s]);
            }
        }
        commit(&bars[7]);
        while (!mtry(&bars[7], 0)) {
        }
        cyc[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 8 * 1024);
    unsigned long long h[1024];
    const char* names[] = {"MMAs only", "+1 commit", "+fence::after", "+mbarrier wait", "+2nd commit", "elect+waits+commits", "elect MMAs only", "elect unrolled 5", "-", "-"};
    for (int nkb = 4; nkb <= 5; ++nkb)
        for (int v = 0; v < 8; ++v) {
            const int iters = 4000;
            k<<<sms, 128>>>(iters, v, nkb, cyc);
            if (cudaDeviceSynchronize() != cudaSuccess) { printf("err %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
            cudaMemcpy(h, cyc, 8 * sms, cudaMemcpyDeviceToHost);
            double m = 0;
            for (int i = 0; i < sms; ++i) m += h[i];
            m /= sms;
            printf("%d MMAs/group %-16s: %.1f cycles per group (%.1f per MMA)\n", nkb, names[v], m / iters, m / iters / nkb);
        }
    return 0;
}
