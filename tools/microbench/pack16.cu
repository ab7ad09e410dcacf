// pack16.cu -- checks the semantics of tcgen05.ld .pack::16b on B200: which
// 16 bits of two adjacent 32-bit TMEM columns land in one register.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void k(uint32_t* out) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + (uint32_t(warp * 32) << 16);
    if (warp == 0) {
        // column c of lane `lane` holds 0xC0DE0000 + (lane << 8) + c  (high half marker, low half = lane,col)
        uint32_t v[4];
        for (int c = 0; c < 4; ++c) v[c] = 0xC0DE0000u + (uint32_t(lane) << 8) + uint32_t(c);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(base), "r"(v[0]), "r"(v[1]),
                     "r"(v[2]), "r"(v[3]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        uint32_t r0, r1;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.pack::16b.b32 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(base));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        out[lane * 2] = r0;
        out[lane * 2 + 1] = r1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(slot));
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 64 * 4);
    k<<<1, 32>>>(d);
    uint32_t h[64];
    if (cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost) != cudaSuccess) { printf("error %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
    for (int l = 0; l < 3; ++l) printf("lane %d: r0=%08x r1=%08x   (columns hold c0de%02x00..03)\n", l, h[2 * l], h[2 * l + 1], l);
    return 0;
}
