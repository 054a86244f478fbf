// Dependent-chain latency of FFMA vs FFMA2 (one warp), cycles per instruction.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__global__ void lat_ffma(float* out, long long* cyc, float a, float b) {
  float x = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 128
  for (int i = 0; i < 4096; i++) x = fmaf(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_ffma2(float* out, long long* cyc, float a, float b) {
  u64 x = (u64)__float_as_uint((float)threadIdx.x) | ((u64)__float_as_uint(1.f) << 32);
  u64 A = (u64)__float_as_uint(a) | ((u64)__float_as_uint(a) << 32);
  u64 B = (u64)__float_as_uint(b) | ((u64)__float_as_uint(b) << 32);
  long long t0 = clock64();
#pragma unroll 128
  for (int i = 0; i < 4096; i++) x = f2fma(x, A, B);
  long long t1 = clock64();
  out[threadIdx.x] = __uint_as_float((unsigned)x) + __uint_as_float((unsigned)(x >> 32)); if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 4096); cudaMallocManaged(&cyc, 8);
  lat_ffma<<<1, 32>>>(out, cyc, 0.999f, 0.5f); cudaDeviceSynchronize();
  lat_ffma<<<1, 32>>>(out, cyc, 0.999f, 0.5f); cudaDeviceSynchronize();
  printf("FFMA  dependent latency: %.2f cycles\n", cyc[0] / 4096.0);
  lat_ffma2<<<1, 32>>>(out, cyc, 0.999f, 0.5f); cudaDeviceSynchronize();
  lat_ffma2<<<1, 32>>>(out, cyc, 0.999f, 0.5f); cudaDeviceSynchronize();
  printf("FFMA2 dependent latency: %.2f cycles\n", cyc[0] / 4096.0);
  return 0;
}
