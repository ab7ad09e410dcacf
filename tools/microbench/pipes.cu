// Pipe-throughput microbenchmarks used to choose the scan kernel's design
// (POPC vs legacy IMMA vs ALU expansion vs HBM streaming). Not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_popc(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
  uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      s0 += __popc(a ^ (s1 + j)); s1 += __popc(b ^ (s2 + j)); s2 += __popc(c ^ (s3 + j)); s3 += __popc(d ^ (s0 + j));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}

__global__ void k_lop(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t a = in[threadIdx.x], b = in[threadIdx.x + 1], c = in[threadIdx.x + 2], d = in[threadIdx.x + 3];
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a = (a >> 3) & 0x07070707u ^ b; b = (b >> 5) & 0x03030303u ^ c; c = (c << 1) & 0x06060606u ^ d; d = (d >> 7) & 0x01010101u ^ a;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

__global__ void k_isetp(const int* in, int* out, int iters) {
  int a[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = in[threadIdx.x + j];
  int t = in[0];
  unsigned hit = 0;
  for (int i = 0; i < iters; ++i) {
    bool p = false;
#pragma unroll
    for (int j = 0; j < 16; ++j) p |= (a[j] >= t + i);
    hit += p;
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] ^= i;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = hit;
}

__global__ void k_imma(const int* in, int* out, int iters) {
  uint32_t a0 = in[threadIdx.x], a1 = in[threadIdx.x + 1], a2 = in[threadIdx.x + 2], a3 = in[threadIdx.x + 3];
  uint32_t b0 = in[threadIdx.x + 4], b1 = in[threadIdx.x + 5];
  int c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  int s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dd(const double* in, double* out, int iters) {
  double a = in[threadIdx.x], b = in[threadIdx.x + 1] + 3.0, c = in[threadIdx.x + 2] + 5.0, d = in[threadIdx.x + 3] + 7.0;
  double s = 0;
  for (int i = 0; i < iters; ++i) {
    s += __ddiv_rn(a + i, b); s += __ddiv_rn(c + i, d);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_read(const uint4* __restrict__ in, size_t n, uint32_t* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(in + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("sms=%d clock_khz=%d\n", sms, clk);
  uint32_t* buf; CK(cudaMalloc(&buf, 1 << 20)); CK(cudaMemset(buf, 1, 1 << 20));
  uint32_t* out; CK(cudaMalloc(&out, 64 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid = sms * 8, block = 256, iters = 2000;
  float ms;
  auto tm = [&](auto launch, double ops, const char* name) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-8s %8.3f ms  %10.3f Gop/s  %8.2f op/clk/SM(at %d MHz)\n", name, ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  };
  double nthreads = (double)grid * block;
  tm([&] { k_popc<<<grid, block>>>(buf, out, iters); }, nthreads * iters * 64, "popc");
  tm([&] { k_lop<<<grid, block>>>(buf, out, iters); }, nthreads * iters * 16 * 4 * 3, "shf/lop");
  tm([&] { k_isetp<<<grid, block>>>((int*)buf, (int*)out, iters); }, nthreads * iters * 16, "isetp");
  // IMMA: m16n8k32 = 4096 MAC per warp-instruction
  tm([&] { k_imma<<<grid, block>>>((int*)buf, (int*)out, iters); }, nthreads / 32 * iters * 8 * 4096.0 * 2, "imma");
  tm([&] { k_dd<<<grid, block>>>((double*)buf, (double*)out, iters); }, nthreads * iters * 2, "ddiv");
  size_t bytes = (size_t)8 << 30; uint4* big; CK(cudaMalloc(&big, bytes)); CK(cudaMemset(big, 3, bytes));
  for (int occ : {4, 8, 16}) {
    tm([&] { k_read<<<sms * occ, 512>>>(big, bytes / 16, out); }, (double)bytes, occ == 4 ? "read4" : occ == 8 ? "read8" : "read16");
  }
  printf("(read: Gop/s == GB/s)\n");
  return 0;
}
