// Microbenchmark: FFMA vs FFMA2 (fma.rn.f32x2) issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ffma(float *out, int iters, float a, float b) {
  float r[16];
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fmaf(r[i], a, b);
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long x, unsigned long long y, unsigned long long z) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(x), "l"(y), "l"(z));
  return d;
}
__global__ void k_ffma2(float *out, int iters, float a, float b) {
  unsigned long long r[16];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *reinterpret_cast<unsigned long long *>(&av), B = *reinterpret_cast<unsigned long long *>(&bv);
  for (int i = 0; i < 16; ++i) { float2 t = make_float2(threadIdx.x * 0.001f + i, i * 0.5f); r[i] = *reinterpret_cast<unsigned long long *>(&t); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = ffma2(r[i], A, B);
  }
  float s = 0; for (int i = 0; i < 16; ++i) { float2 t = *reinterpret_cast<float2 *>(&r[i]); s += t.x + t.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float *o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int iters = 20000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    for (int warps = 4; warps <= 32; warps *= 2) {
      float ms1, ms2;
      cudaEventRecord(e0); k_ffma<<<148, 32 * warps>>>(o, iters, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms1, e0, e1);
      cudaEventRecord(e0); k_ffma2<<<148, 32 * warps>>>(o, iters, 0.999f, 0.001f); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms2, e0, e1);
      double fl = 148.0 * 32 * warps * iters * 16;   // FMA per kernel (ffma); ffma2 does 2x
      if (rep) printf("warps/SM %2d  FFMA %.1f TFMA/s   FFMA2 %.1f TFMA/s\n", warps, fl / ms1 / 1e9, 2 * fl / ms2 / 1e9);
    }
  }
  return 0;
}
