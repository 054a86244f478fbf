// Microbenchmark: packed FP32x2 FMA (FFMA2, sm_100a) throughput for the lattice's operand forms.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
#define CH 8
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 pack(float x, float y) {
  return (u64)__float_as_uint(x) | ((u64)__float_as_uint(y) << 32);
}
__device__ __forceinline__ float lo(u64 v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi(u64 v) { return __uint_as_float((unsigned)(v >> 32)); }

__global__ void k_reg3(float* out, float s) {
  u64 x[CH], y[CH], z[CH];
  for (int c = 0; c < CH; c++) { x[c] = pack(threadIdx.x * 1e-3f + c, c); y[c] = pack(s + c * 1e-4f, s); z[c] = pack(s * 0.5f + c, 1.f); }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = f2fma(x[c], y[c], z[c]);
  }
  float r = 0; for (int c = 0; c < CH; c++) r += lo(x[c]) + hi(x[c]);
  if (r == 1234.5f) out[threadIdx.x] = r;
}
__global__ void k_uni(float* out, float s, float cc) {
  u64 x[CH], z[CH];
  const u64 c2 = pack(cc, cc);
  for (int c = 0; c < CH; c++) { x[c] = pack(threadIdx.x * 1e-3f + c, c); z[c] = pack(s * 0.5f + c, 1.f); }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = f2fma(x[c], c2, z[c]);
  }
  float r = 0; for (int c = 0; c < CH; c++) r += lo(x[c]) + hi(x[c]);
  if (r == 1234.5f) out[threadIdx.x] = r;
}
// lattice cell on two windows at once: u = Q*f[e] + f[e+1]; v = a*prev + u
__global__ void k_cell2x(float* out, float s, float a) {
  u64 q[16], f[16];
  const u64 a2 = pack(a, a);
  for (int c = 0; c < 16; c++) { q[c] = pack(s + c * 1e-3f, s); f[c] = pack(threadIdx.x * 1e-4f + c, c); }
  for (int it = 0; it < ITERS / 4; it++) {
    u64 prev = 0ull;
#pragma unroll
    for (int e = 0; e < 15; e++) {
      u64 u = f2fma(q[e], f[e], f[e + 1]);
      u64 v = f2fma(a2, prev, u);
      f[e] = v; prev = v;
    }
  }
  float r = 0; for (int c = 0; c < 16; c++) r += lo(f[c]) + hi(f[c]);
  if (r == 1234.5f) out[threadIdx.x] = r;
}
// two pairs interleaved (4 windows per lane)
__global__ void k_cell4x(float* out, float s, float a) {
  u64 q[16], f[16], g[16];
  const u64 a2 = pack(a, a);
  for (int c = 0; c < 16; c++) { q[c] = pack(s + c * 1e-3f, s); f[c] = pack(threadIdx.x * 1e-4f + c, c); g[c] = pack(c, 1.f); }
  for (int it = 0; it < ITERS / 8; it++) {
    u64 p1 = 0ull, p2 = 0ull;
#pragma unroll
    for (int e = 0; e < 15; e++) {
      u64 u = f2fma(q[e], f[e], f[e + 1]);
      u64 w = f2fma(q[e], g[e], g[e + 1]);
      u64 v = f2fma(a2, p1, u);
      u64 x = f2fma(a2, p2, w);
      f[e] = v; p1 = v; g[e] = x; p2 = x;
    }
  }
  float r = 0; for (int c = 0; c < 16; c++) r += lo(f[c]) + hi(f[c]) + lo(g[c]);
  if (r == 1234.5f) out[threadIdx.x] = r;
}
int main() {
  float* out; cudaMalloc(&out, 4096);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int threads : {128, 256}) for (int bps : {4, 8}) {
    dim3 grid(sms * bps), block(threads);
    double nthr = (double)grid.x * threads;
    auto run = [&](const char* name, auto launch, double fma_per_thread) {
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(a); for (int r = 0; r < 5; r++) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("threads=%d blocks/SM=%d %-8s %.2f TFLOP/s (scalar-FMA rate)  err=%s\n", threads, bps, name,
             5 * nthr * fma_per_thread * 2 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    };
    run("f2reg3", [&] { k_reg3<<<grid, block>>>(out, 1.0f); }, (double)ITERS * CH * 2);
    run("f2uni", [&] { k_uni<<<grid, block>>>(out, 1.0f, 0.999f); }, (double)ITERS * CH * 2);
    run("cell2x", [&] { k_cell2x<<<grid, block>>>(out, 1.0f, 0.005f); }, (double)(ITERS / 4) * 30 * 2);
    run("cell4x", [&] { k_cell4x<<<grid, block>>>(out, 1.0f, 0.005f); }, (double)(ITERS / 8) * 60 * 2);
  }
  return 0;
}
