// Microbenchmark: cost of the per-row warp-uniform table dispatch in the lattice (B200).
// Build: python tools/ubench/gen_brx.py && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dispatch dispatch.cu
// Measured (warps/SM 12-20, fraction of the FMA pipe): nodisp 0.75, disp2 0.55, disp1 0.51, select 0.50,
// disp3 0.49, pred 0.25, brx.idx jump tables 0.36-0.46.
// A "lattice" = NR rows of MN nodes on two windows (FFMA2); row r uses table q1 or q0 by bit r
// of a per-lattice codeword x that is warp-uniform (read from shared memory per lattice).
//   k_nodisp : rows always use q1 (no branch) -- the ceiling
//   k_disp1  : one 2-way uniform branch per row
//   k_disp2  : one 4-way switch per row pair
//   k_sel    : branch-free, Q = x_r ? q1 : q0 per node pair via selects
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 pack(float x, float y) { return (u64)__float_as_uint(x) | ((u64)__float_as_uint(y) << 32); }
__device__ __forceinline__ float lo(u64 v) { return __uint_as_float((unsigned)v); }
#define MN 14
#define NR 9
#define JJ (NR + MN + 2)
#define NLAT 256
#include "brx_rows.cuh"
// u = (x_r ? q1 : q0) * f + g as two predicated FFMA2 (no branch, no select)
__device__ __forceinline__ u64 f2fma_pred(uint32_t bit, u64 q1, u64 q0, u64 b, u64 c) {
  u64 d;
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
      "@p fma.rn.f32x2 %0, %2, %4, %5;\n\t@!p fma.rn.f32x2 %0, %3, %4, %5;\n\t}"
      : "=l"(d) : "r"(bit), "l"(q1), "l"(q0), "l"(b), "l"(c));
  return d;
}
template <int MODE>
__device__ __forceinline__ void lrow(u64 (&f)[MN], const u64 (&q1)[JJ], const u64 (&q0)[JJ], int r, uint32_t x, u64 a2, bool b) {
  u64 prev = 0ull;
#pragma unroll
  for (int e = 0; e < MN; e++) {
    u64 u;
    if (MODE == 4) {
      u = f2fma_pred((x >> r) & 1u, q1[r + e], q0[r + e], f[e], (e + 1 < MN) ? f[e + 1] : 0ull);
    } else {
      u64 Q;
      if (MODE == 3) Q = ((x >> r) & 1u) ? q1[r + e] : q0[r + e];
      else Q = b ? q1[r + e] : q0[r + e];
      u = (e + 1 < MN) ? f2fma(Q, f[e], f[e + 1]) : f2fma(Q, f[e], 0ull);
    }
    const u64 v = e > 0 ? f2fma(a2, prev, u) : u;
    f[e] = v; prev = v;
  }
}
template <int MODE>
__global__ void k_lat(float* out, const uint32_t* xs, float s, float a) {
  __shared__ uint32_t sx[NLAT];
  for (int t = threadIdx.x; t < NLAT; t += blockDim.x) sx[t] = xs[t];
  __syncthreads();
  u64 q1[JJ], q0[JJ];
  for (int c = 0; c < JJ; c++) { q1[c] = pack(s + c * 1e-3f + threadIdx.x * 1e-7f, s); q0[c] = pack(s * 0.5f, s + c * 1e-4f); }
  const u64 a2 = pack(a, a);
  u64 acc[MN];
  for (int e = 0; e < MN; e++) acc[e] = 0ull;
  for (int l = 0; l < NLAT; l++) {
    const uint32_t x = sx[l];
    u64 f[MN];
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = pack(1.f + e, __uint_as_float(x & 0x3fffffffu) * 1e-30f + 1.f);  // depends on x: not hoistable
    if (MODE == 0) {
#pragma unroll
      for (int r = 0; r < NR; r++) lrow<0>(f, q1, q0, r, x, a2, true);
    } else if (MODE == 1) {
#pragma unroll
      for (int r = 0; r < NR; r++) {
        if ((x >> r) & 1u) lrow<1>(f, q1, q0, r, x, a2, true);
        else lrow<1>(f, q1, q0, r, x, a2, false);
      }
    } else if (MODE == 2) {
#pragma unroll
      for (int r = 0; r + 1 < NR; r += 2) {
        switch ((x >> r) & 3u) {
          case 0: lrow<2>(f, q1, q0, r, x, a2, false); lrow<2>(f, q1, q0, r + 1, x, a2, false); break;
          case 1: lrow<2>(f, q1, q0, r, x, a2, true); lrow<2>(f, q1, q0, r + 1, x, a2, false); break;
          case 2: lrow<2>(f, q1, q0, r, x, a2, false); lrow<2>(f, q1, q0, r + 1, x, a2, true); break;
          default: lrow<2>(f, q1, q0, r, x, a2, true); lrow<2>(f, q1, q0, r + 1, x, a2, true); break;
        }
      }
      if (NR & 1) {
        if ((x >> (NR - 1)) & 1u) lrow<2>(f, q1, q0, NR - 1, x, a2, true);
        else lrow<2>(f, q1, q0, NR - 1, x, a2, false);
      }
    } else if (MODE == 5) {  // 8-way switch per row triple
#pragma unroll
      for (int r = 0; r + 2 < NR; r += 3) {
        switch ((x >> r) & 7u) {
          case 0: lrow<2>(f, q1, q0, r, x, a2, false); lrow<2>(f, q1, q0, r + 1, x, a2, false); lrow<2>(f, q1, q0, r + 2, x, a2, false); break;
          case 1: lrow<2>(f, q1, q0, r, x, a2, true); lrow<2>(f, q1, q0, r + 1, x, a2, false); lrow<2>(f, q1, q0, r + 2, x, a2, false); break;
          case 2: lrow<2>(f, q1, q0, r, x, a2, false); lrow<2>(f, q1, q0, r + 1, x, a2, true); lrow<2>(f, q1, q0, r + 2, x, a2, false); break;
          case 3: lrow<2>(f, q1, q0, r, x, a2, true); lrow<2>(f, q1, q0, r + 1, x, a2, true); lrow<2>(f, q1, q0, r + 2, x, a2, false); break;
          case 4: lrow<2>(f, q1, q0, r, x, a2, false); lrow<2>(f, q1, q0, r + 1, x, a2, false); lrow<2>(f, q1, q0, r + 2, x, a2, true); break;
          case 5: lrow<2>(f, q1, q0, r, x, a2, true); lrow<2>(f, q1, q0, r + 1, x, a2, false); lrow<2>(f, q1, q0, r + 2, x, a2, true); break;
          case 6: lrow<2>(f, q1, q0, r, x, a2, false); lrow<2>(f, q1, q0, r + 1, x, a2, true); lrow<2>(f, q1, q0, r + 2, x, a2, true); break;
          default: lrow<2>(f, q1, q0, r, x, a2, true); lrow<2>(f, q1, q0, r + 1, x, a2, true); lrow<2>(f, q1, q0, r + 2, x, a2, true); break;
        }
      }
    } else if (MODE >= 6 && MODE <= 8) {  // one indexed jump (brx.idx) per group of G = MODE - 5 rows
      constexpr int G = MODE - 5;
#pragma unroll
      for (int r = 0; r + G <= NR; r += G) brx_rows<G>(f, q1, q0, r, (x >> r) & ((1u << G) - 1u), a2);
#pragma unroll
      for (int r = (NR / G) * G; r < NR; r++) brx_rows<1>(f, q1, q0, r, (x >> r) & 1u, a2);
    } else if (MODE == 3) {
#pragma unroll
      for (int r = 0; r < NR; r++) lrow<3>(f, q1, q0, r, x, a2, true);
    } else {
#pragma unroll
      for (int r = 0; r < NR; r++) lrow<4>(f, q1, q0, r, x, a2, true);
    }
#pragma unroll
    for (int e = 0; e < MN; e++) acc[e] = f2fma(f[e], q1[e], acc[e]);
  }
  float r = 0; for (int e = 0; e < MN; e++) r += lo(acc[e]);
  if (r == 1234.5f) out[threadIdx.x] = r;
}
int main() {
  float* out; cudaMalloc(&out, 1 << 16);
  uint32_t* xs; cudaMalloc(&xs, NLAT * 4);
  uint32_t hx[NLAT]; unsigned st = 12345;
  for (int i = 0; i < NLAT; i++) { st = st * 1103515245u + 12345u; hx[i] = st >> 8; }
  cudaMemcpy(xs, hx, sizeof hx, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double nodes = NR * MN, ffma2 = nodes * 2 + MN;
  for (int bps : {3, 4, 5}) {
    dim3 grid(sms * bps * 4), block(128);
    const double nthr = (double)grid.x * 128;
    auto run = [&](const char* name, auto launch) {
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(a); for (int r = 0; r < 3; r++) launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double tf = 3 * nthr * NLAT * ffma2 * 4 / (ms * 1e-3) / 1e12;
      printf("CTAs/SM=%d %-8s %6.2f TFLOP/s executed (%.3f of 74.45) %s\n", bps, name, tf, tf / 74.45, cudaGetErrorString(cudaGetLastError()));
    };
    run("nodisp", [&] { k_lat<0><<<grid, block>>>(out, xs, 1.0f, 0.005f); });
    run("disp1", [&] { k_lat<1><<<grid, block>>>(out, xs, 1.0f, 0.005f); });
    run("disp2", [&] { k_lat<2><<<grid, block>>>(out, xs, 1.0f, 0.005f); });
    run("select", [&] { k_lat<3><<<grid, block>>>(out, xs, 1.0f, 0.005f); });
    run("disp3", [&] { k_lat<5><<<grid, block>>>(out, xs, 1.0f, 0.005f); });
    run("brx1", [&] { k_lat<6><<<grid, block>>>(out, xs, 1.0f, 0.005f); });
    run("brx2", [&] { k_lat<7><<<grid, block>>>(out, xs, 1.0f, 0.005f); });
    run("brx3", [&] { k_lat<8><<<grid, block>>>(out, xs, 1.0f, 0.005f); });
  }
  return 0;
}
