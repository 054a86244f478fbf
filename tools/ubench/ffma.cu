// Microbenchmark: FP32 FFMA throughput on B200 for operand forms relevant to the lattice.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
#define CH 8
__global__ void k_reg3(float* out, float s) {  // x = x*y + z, y,z distinct registers per chain
  float x[CH], y[CH], z[CH];
  for (int c = 0; c < CH; c++) { x[c] = threadIdx.x * 1e-3f + c; y[c] = s + c * 1e-4f; z[c] = s * 0.5f + c; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = fmaf(x[c], y[c], z[c]);
  }
  float r = 0; for (int c = 0; c < CH; c++) r += x[c];
  if (r == 1234.5f) out[threadIdx.x] = r;
}
__global__ void k_const(float* out, float s, float cc) {  // x = x*c + z, c kernel param
  float x[CH], z[CH];
  for (int c = 0; c < CH; c++) { x[c] = threadIdx.x * 1e-3f + c; z[c] = s * 0.5f + c; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = fmaf(x[c], cc, z[c]);
  }
  float r = 0; for (int c = 0; c < CH; c++) r += x[c];
  if (r == 1234.5f) out[threadIdx.x] = r;
}
__global__ void k_imm(float* out, float s) {
  float x[CH], z[CH];
  for (int c = 0; c < CH; c++) { x[c] = threadIdx.x * 1e-3f + c; z[c] = s * 0.5f + c; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = fmaf(x[c], 0.999f, z[c]);
  }
  float r = 0; for (int c = 0; c < CH; c++) r += x[c];
  if (r == 1234.5f) out[threadIdx.x] = r;
}
// lattice-like: per cell u = q*f + g (3 regs), chain v = a*v + u (a const)
__global__ void k_cell(float* out, float s, float a) {
  float q[16], f[16];
  for (int c = 0; c < 16; c++) { q[c] = s + c * 1e-3f; f[c] = threadIdx.x * 1e-4f + c; }
  for (int it = 0; it < ITERS / 4; it++) {
    float prev = 0.f;
#pragma unroll
    for (int e = 0; e < 15; e++) {
      float u = fmaf(q[e], f[e], f[e + 1]);
      float v = fmaf(a, prev, u);
      f[e] = v; prev = v;
    }
  }
  float r = 0; for (int c = 0; c < 16; c++) r += f[c];
  if (r == 1234.5f) out[threadIdx.x] = r;
}
// same with two interleaved independent lattices (ILP 2)
__global__ void k_cell2(float* out, float s, float a) {
  float q[16], f[16], g[16];
  for (int c = 0; c < 16; c++) { q[c] = s + c * 1e-3f; f[c] = threadIdx.x * 1e-4f + c; g[c] = f[c] * 0.5f; }
  for (int it = 0; it < ITERS / 8; it++) {
    float p1 = 0.f, p2 = 0.f;
#pragma unroll
    for (int e = 0; e < 15; e++) {
      float u = fmaf(q[e], f[e], f[e + 1]);
      float w = fmaf(q[e], g[e], g[e + 1]);
      float v = fmaf(a, p1, u);
      float x = fmaf(a, p2, w);
      f[e] = v; p1 = v; g[e] = x; p2 = x;
    }
  }
  float r = 0; for (int c = 0; c < 16; c++) r += f[c] + g[c];
  if (r == 1234.5f) out[threadIdx.x] = r;
}
// predicated formulation (Ps = 0): t = a*prev + f[e+1]; @match t += c*f[e]
__global__ void k_pred(float* out, float s, float a, float cq, unsigned mask0) {
  float f[16];
  unsigned m = mask0 ^ (threadIdx.x * 2654435761u);
  for (int c = 0; c < 16; c++) f[c] = threadIdx.x * 1e-4f + c;
  for (int it = 0; it < ITERS / 4; it++) {
    float prev = 0.f;
    unsigned mm = m >> (it & 7);
#pragma unroll
    for (int e = 0; e < 15; e++) {
      float t = fmaf(a, prev, f[e + 1]);
      if ((mm >> e) & 1u) t = fmaf(cq, f[e], t);
      f[e] = t; prev = t;
    }
  }
  float r = 0; for (int c = 0; c < 16; c++) r += f[c];
  if (r == 1234.5f) out[threadIdx.x] = r;
}
int main() {
  float* out; cudaMalloc(&out, 4096);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int threads : {256, 512}) for (int bps : {4, 8}) {
    dim3 grid(sms * bps), block(threads);
    double nthr = (double)grid.x * threads;
    auto run = [&](const char* name, auto launch, double ffma_per_thread) {
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(a); for (int r = 0; r < 5; r++) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double tf = 5 * nthr * ffma_per_thread * 2 / (ms * 1e-3) / 1e12;
      printf("threads=%d blocks/SM=%d %-8s %.2f TFLOP/s (FFMA-rate)\n", threads, bps, name, tf);
    };
    run("reg3", [&] { k_reg3<<<grid, block>>>(out, 1.0f); }, (double)ITERS * CH);
    run("const", [&] { k_const<<<grid, block>>>(out, 1.0f, 0.999f); }, (double)ITERS * CH);
    run("imm", [&] { k_imm<<<grid, block>>>(out, 1.0f); }, (double)ITERS * CH);
    run("cell", [&] { k_cell<<<grid, block>>>(out, 1.0f, 0.005f); }, (double)(ITERS / 4) * 30);
    run("cell2", [&] { k_cell2<<<grid, block>>>(out, 1.0f, 0.005f); }, (double)(ITERS / 8) * 60);
    run("pred", [&] { k_pred<<<grid, block>>>(out, 1.0f, 0.005f, 98.f, 0x5a5a5a5au); }, (double)(ITERS / 4) * 30);
  }
  return 0;
}
