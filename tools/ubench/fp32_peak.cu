// Measured FP32 / FP64 FMA-pipe peaks of this B200 (the ALU roofline denominators of bench.py).
// Independent chains (no dependency stalls), every SM busy (8 CTAs x 256 threads per SM), best of
// 10 launches timed with CUDA events.  Prints one JSON object:
//   ffma2_tflops   : fma.rn.f32x2 (FFMA2), 4 flop per instruction per thread, register operands
//   ffma_tflops    : scalar FFMA with one uniform operand (the scalar FFMA's fastest form)
//   dfma_tflops    : DFMA
// The SM clock is sampled outside (nvidia-smi, tools/gpu_r02.sh): clock64 cycles over the event time
// came out at ~1466 MHz while nvidia-smi read 1965 MHz under load, so it is not reported.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 8192
#define CH 8
typedef unsigned long long u64;

__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 pack(float x, float y) {
  return (u64)__float_as_uint(x) | ((u64)__float_as_uint(y) << 32);
}

__global__ void k_ffma2(float* out, long long* cyc, float s) {
  u64 x[CH], y[CH], z[CH];
  for (int c = 0; c < CH; c++) {
    x[c] = pack(threadIdx.x * 1e-3f + c, c);
    y[c] = pack(s + c * 1e-4f, s);
    z[c] = pack(s * 0.5f + c, 1.f);
  }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = f2fma(x[c], y[c], z[c]);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float r = 0;
  for (int c = 0; c < CH; c++) r += __uint_as_float((unsigned)x[c]) + __uint_as_float((unsigned)(x[c] >> 32));
  if (r == 1234.5f) out[threadIdx.x] = r;
}

__global__ void k_ffma(float* out, float s, float u) {
  float x[CH], z[CH];
  for (int c = 0; c < CH; c++) { x[c] = threadIdx.x * 1e-3f + c; z[c] = s * 0.5f + c; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = fmaf(x[c], u, z[c]);
  }
  float r = 0;
  for (int c = 0; c < CH; c++) r += x[c];
  if (r == 1234.5f) out[threadIdx.x] = r;
}

__global__ void k_dfma(double* out, double s, double u) {
  double x[CH], z[CH];
  for (int c = 0; c < CH; c++) { x[c] = threadIdx.x * 1e-3 + c; z[c] = s * 0.5 + c; }
  for (int it = 0; it < ITERS / 8; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = fma(x[c], u, z[c]);
  }
  double r = 0;
  for (int c = 0; c < CH; c++) r += x[c];
  if (r == 1234.5) out[threadIdx.x] = r;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int bps = 8, threads = 256;
  dim3 grid(sms * bps), block(threads);
  cudaMalloc(&cyc, sizeof(long long) * grid.x);
  const double nthr = (double)grid.x * threads;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto best = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    float bestms = 1e30f;
    for (int r = 0; r < 10; r++) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < bestms) bestms = ms;
    }
    return (double)bestms;
  };
  double ms2 = best([&] { k_ffma2<<<grid, block>>>(out, cyc, 1.0f); });
  long long* h = new long long[grid.x];
  cudaMemcpy(h, cyc, sizeof(long long) * grid.x, cudaMemcpyDeviceToHost);
  double cmax = 0;
  for (unsigned i = 0; i < grid.x; i++) cmax = h[i] > cmax ? h[i] : cmax;
  double ms1 = best([&] { k_ffma<<<grid, block>>>(out, 1.0f, 0.999f); });
  double msd = best([&] { k_dfma<<<grid, block>>>((double*)out, 1.0, 0.999); });
  const double f2 = nthr * ITERS * CH * 4 / (ms2 * 1e-3) / 1e12;
  const double f1 = nthr * ITERS * CH * 2 / (ms1 * 1e-3) / 1e12;
  const double fd = nthr * (ITERS / 8) * CH * 2 / (msd * 1e-3) / 1e12;
  (void)cmax;
  printf("{\"sms\": %d, \"ffma2_tflops\": %.3f, \"ffma_tflops\": %.3f, \"dfma_tflops\": %.3f, \"err\": \"%s\"}\n",
         sms, f2, f1, fd, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
