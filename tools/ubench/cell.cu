// Microbenchmark: which part of the lattice node pattern limits FFMA2 throughput on B200.
//   u[e] = Q[e] * f[e] + f[e+1]   (3 register-pair sources, independent across e)
//   v[e] = a * v[e-1] + u[e]      (serial insertion chain along the row)
// Variants isolate the u-part, the chain, the operand forms and the instruction order.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 1024
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 pack(float x, float y) { return (u64)__float_as_uint(x) | ((u64)__float_as_uint(y) << 32); }
__device__ __forceinline__ float lo(u64 v) { return __uint_as_float((unsigned)v); }

#define MN 14
// full node: u then chain, a2 from a register pair
__global__ void k_node_reg(float* out, float s, float a) {
  u64 q[MN], f[MN + 1];
  const u64 a2 = pack(a + threadIdx.x * 1e-9f, a);
  for (int c = 0; c < MN; c++) { q[c] = pack(s + c * 1e-3f, s); f[c] = pack(threadIdx.x * 1e-4f + c, c); }
  f[MN] = 0ull;
  for (int it = 0; it < ITERS; it++) {
    u64 prev = 0ull;
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const u64 u = f2fma(q[e], f[e], f[e + 1]);
      const u64 v = f2fma(a2, prev, u);
      f[e] = v; prev = v;
    }
  }
  float r = 0; for (int c = 0; c < MN; c++) r += lo(f[c]);
  if (r == 1234.5f) out[threadIdx.x] = r;
}
// u-part only (no chain): every FFMA2 independent within the row
__global__ void k_u_only(float* out, float s) {
  u64 q[MN], f[MN + 1];
  for (int c = 0; c < MN; c++) { q[c] = pack(s + c * 1e-3f, s); f[c] = pack(threadIdx.x * 1e-4f + c, c); }
  f[MN] = 0ull;
  for (int it = 0; it < 2 * ITERS; it++) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = f2fma(q[e], f[e], f[e + 1]);
  }
  float r = 0; for (int c = 0; c < MN; c++) r += lo(f[c]);
  if (r == 1234.5f) out[threadIdx.x] = r;
}
// chain only: v = a v + u[e], u from registers (serial, latency-bound per thread)
__global__ void k_chain_only(float* out, float s, float a) {
  u64 u[MN];
  const u64 a2 = pack(a, a);
  for (int c = 0; c < MN; c++) u[c] = pack(s + c * 1e-3f, s + threadIdx.x * 1e-6f);
  u64 v = 0ull;
  for (int it = 0; it < 2 * ITERS; it++) {
#pragma unroll
    for (int e = 0; e < MN; e++) v = f2fma(a2, v, u[e]);
  }
  if (lo(v) == 1234.5f) out[threadIdx.x] = lo(v);
}
// two rows in flight (row r+1 lags row r): the real kernel's row pairs
__global__ void k_node_pairs(float* out, float s, float a) {
  u64 q[MN], q2[MN], f[MN + 1];
  const u64 a2 = pack(a + threadIdx.x * 1e-9f, a);
  for (int c = 0; c < MN; c++) { q[c] = pack(s + c * 1e-3f, s); q2[c] = pack(s, s + c * 1e-3f); f[c] = pack(threadIdx.x * 1e-4f + c, c); }
  f[MN] = 0ull;
  for (int it = 0; it < ITERS / 2; it++) {
    u64 p1 = 0ull, p2 = 0ull;
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const u64 u = f2fma(q[e], f[e], f[e + 1]);
      const u64 v = f2fma(a2, p1, u);
      f[e] = v; p1 = v;
    }
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const u64 u = f2fma(q2[e], f[e], f[e + 1]);
      const u64 v = f2fma(a2, p2, u);
      f[e] = v; p2 = v;
    }
  }
  float r = 0; for (int c = 0; c < MN; c++) r += lo(f[c]);
  if (r == 1234.5f) out[threadIdx.x] = r;
}
// node with the chain product taken first: v = u + a prev written as fma(prev, a, u) (same math)
// but u built from the row's left neighbour to vary register pairing: u = f[e+1] + Q f[e]
__global__ void k_node_swap(float* out, float s, float a) {
  u64 q[MN], f[MN + 1];
  const u64 a2 = pack(a + threadIdx.x * 1e-9f, a);
  for (int c = 0; c < MN; c++) { q[c] = pack(s + c * 1e-3f, s); f[c] = pack(threadIdx.x * 1e-4f + c, c); }
  f[MN] = 0ull;
  for (int it = 0; it < ITERS; it++) {
    u64 prev = 0ull;
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const u64 u = f2fma(f[e], q[e], f[e + 1]);
      const u64 v = f2fma(prev, a2, u);
      f[e] = v; prev = v;
    }
  }
  float r = 0; for (int c = 0; c < MN; c++) r += lo(f[c]);
  if (r == 1234.5f) out[threadIdx.x] = r;
}

int main() {
  float* out; cudaMalloc(&out, 1 << 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int threads : {128, 256}) for (int bps : {2, 3, 4, 8}) {
    dim3 grid(sms * bps), block(threads);
    double nthr = (double)grid.x * threads;
    auto run = [&](const char* name, auto launch, double ffma2_per_thread) {
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(a); for (int r = 0; r < 5; r++) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double tf = 5 * nthr * ffma2_per_thread * 4 / (ms * 1e-3) / 1e12;
      printf("warps/SM=%2d %-10s %6.2f TFLOP/s executed (%.3f of 74.45)  %s\n", threads / 32 * bps, name, tf, tf / 74.45,
             cudaGetErrorString(cudaGetLastError()));
    };
    run("node_reg", [&] { k_node_reg<<<grid, block>>>(out, 1.0f, 0.005f); }, (double)ITERS * MN * 2);
    run("node_swap", [&] { k_node_swap<<<grid, block>>>(out, 1.0f, 0.005f); }, (double)ITERS * MN * 2);
    run("node_pairs", [&] { k_node_pairs<<<grid, block>>>(out, 1.0f, 0.005f); }, (double)ITERS * MN * 2);
    run("u_only", [&] { k_u_only<<<grid, block>>>(out, 1.0f); }, (double)2 * ITERS * MN);
    run("chain_only", [&] { k_chain_only<<<grid, block>>>(out, 1.0f, 0.005f); }, (double)2 * ITERS * MN);
  }
  return 0;
}
