// Microbenchmark: issue / pipe throughput of FFMA vs FFMA2 vs FADD2 on sm_100a,
// and a mix with shared-memory loads.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d; asm volatile("fma.rn.f32x2 %0,%1,%2,%3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 d; asm volatile("add.rn.f32x2 %0,%1,%2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float fma1(float a, float b, float c) {
  float d; asm volatile("fma.rn.f32 %0,%1,%2,%3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ unsigned iadd(unsigned a, unsigned b) {
  unsigned d; asm volatile("add.u32 %0,%1,%2;" : "=r"(d) : "r"(a), "r"(b)); return d; }

template <int MODE>
__global__ void k(float* out, int iters, float s) {
  constexpr int C = 8;
  u64 v[C]; float f[C]; unsigned u[C];
  for (int i = 0; i < C; ++i) { v[i] = threadIdx.x + i; f[i] = threadIdx.x * 0.5f + i; u[i] = threadIdx.x + i; }
  u64 b = __float_as_uint(s) | (u64(__float_as_uint(s)) << 32);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) {
      if (MODE == 0) f[i] = fma1(f[i], s, f[i]);
      if (MODE == 1) v[i] = fma2(v[i], b, v[i]);
      if (MODE == 2) v[i] = add2(v[i], b);
      if (MODE == 3) { v[i] = fma2(v[i], b, v[i]); u[i] = iadd(u[i], 3u); }   // FFMA2 + IADD
      if (MODE == 4) { f[i] = fma1(f[i], s, f[i]); u[i] = iadd(u[i], 3u); }   // FFMA + IADD
      if (MODE == 5) { v[i] = fma2(v[i], b, v[i]); f[i] = fma1(f[i], s, f[i]); } // FFMA2 + FFMA
    }
  }
  float acc = 0;
  for (int i = 0; i < C; ++i) acc += f[i] + __uint_as_float(unsigned(v[i])) + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 1024 * sizeof(float));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096, threads = 512, blocks = 148 * 4;
  const char* names[] = {"FFMA", "FFMA2", "FADD2", "FFMA2+IADD", "FFMA+IADD", "FFMA2+FFMA"};
  for (int m = 0; m < 6; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (m) {
        case 0: k<0><<<blocks, threads>>>(d, iters, 1.0001f); break;
        case 1: k<1><<<blocks, threads>>>(d, iters, 1.0001f); break;
        case 2: k<2><<<blocks, threads>>>(d, iters, 1.0001f); break;
        case 3: k<3><<<blocks, threads>>>(d, iters, 1.0001f); break;
        case 4: k<4><<<blocks, threads>>>(d, iters, 1.0001f); break;
        case 5: k<5><<<blocks, threads>>>(d, iters, 1.0001f); break;
      }
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) {
        double warp_insts = double(blocks) * threads / 32 * iters * 8 * (m >= 3 ? 2 : 1);
        double per_smsp_per_ns = warp_insts / (148.0 * 4) / (ms * 1e6);
        printf("%-12s %8.3f ms  %.3f warp-inst/ns/SMSP (clock attr %d kHz)\n", names[m], ms, per_smsp_per_ns, clk);
      }
    }
  }
  return 0;
}
