// k_alphabeta_warp.cuh -- a2/a3 for small trellises (M_tau <= 128): one warp per
// (frame, direction), SPT = ceil(M_tau / 32) states per lane, no block barrier.
//
//   alpha'_{i+1}(m) = sum_k alpha_i(m - k) Gamma_i(m - k, k)      (eqn:alpha_prenorm)
//   beta'_i(m')     = sum_k Gamma_i(m', k) beta_{i+1}(m' + k)     (eqn:beta)
// then division by the row sum (eqn:alpha_norm; "similar" for beta), FP64.
// The row lives in this warp's shared-memory slice; Gamma_i is read straight from
// HBM/L2 (M_n coalesced loads per state), latency hidden by the many resident warps.
#pragma once
#include "common.cuh"

namespace bsidmap {

constexpr int kAbWarpThreads = 256;  // 8 (frame, direction) tasks per CTA

template <int SPT, int MN>
__global__ void __launch_bounds__(kAbWarpThreads, 2) k_alpha_beta_warp(const DecodeParams p) {
  extern __shared__ __align__(16) double s_rows[];  // [8][SPT * 32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long task = (long)blockIdx.x * (kAbWarpThreads / 32) + warp;
  if (task >= 2L * p.F) return;  // warp-uniform
  const int f = (int)(task >> 1);
  const bool fwd = (task & 1) == 0;
  if (p.status[f] != kFrameOk) return;
  const int Mt = p.Mt, N = p.N, lo = p.mn_lo;
  double* row = s_rows + warp * SPT * 32;
  double* rows_g = (fwd ? p.alpha : p.beta) + (size_t)f * (N + 1) * Mt;
  const float* Gf = p.Gsum + (size_t)f * N * MN * Mt;
  const int boundary = fwd ? -p.mt_lo : p.rho[f] - p.n * N - p.mt_lo;  // alpha_0 = delta(0), beta_N = delta(rho - tau)
  const int i0 = fwd ? 0 : N;
#pragma unroll
  for (int s = 0; s < SPT; s++) {
    const int m = lane + 32 * s;
    const double v = (m == boundary) ? 1.0 : 0.0;
    row[m] = v;
    if (m < Mt) rows_g[(size_t)i0 * Mt + m] = v;
  }
  __syncwarp();
  for (int step = 0; step < N; step++) {
    const int i = fwd ? step : N - 1 - step;
    const float* G = Gf + (size_t)i * MN * Mt;  // [k][m']
    // all SPT * M_n loads of Gamma_i first (unconditional, clamped addresses) so they are in
    // flight together: one memory latency per step
    float g[SPT][MN];
#pragma unroll
    for (int s = 0; s < SPT; s++) {
      const int m = lane + 32 * s;
#pragma unroll
      for (int e = 0; e < MN; e++) {
        const int idx = fwd ? m - lo - e : m;
        g[s][e] = __ldg(G + (size_t)e * Mt + min(max(idx, 0), Mt - 1));
      }
    }
    double acc[SPT];
    double part = 0.0;
#pragma unroll
    for (int s = 0; s < SPT; s++) {
      const int m = lane + 32 * s;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int e = 0; e < MN; e++) {
        const int idx = fwd ? m - lo - e : m;         // Gamma_i column read by this term
        const int j = fwd ? m - lo - e : m + lo + e;  // neighbouring state of the previous row
        const bool ok = m < Mt && idx >= 0 && idx < Mt && j >= 0 && j < Mt;
        const double r = ok ? row[j] : 0.0;
        const double gv = ok ? (double)g[s][e] : 0.0;
        if (e & 1) a1 = fma(r, gv, a1); else a0 = fma(r, gv, a0);
      }
      acc[s] = a0 + a1;
      part += acc[s];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (!(part > 0.0)) {  // all-zero row: Y impossible under the limits (reading R14)
      if (lane == 0) p.status[f] = kFrameUnderflow;
      return;
    }
    const double inv = 1.0 / part;
    const int r = fwd ? i + 1 : i;
    __syncwarp();
#pragma unroll
    for (int s = 0; s < SPT; s++) {
      const int m = lane + 32 * s;
      const double v = acc[s] * inv;
      row[m] = v;
      if (m < Mt) rows_g[(size_t)r * Mt + m] = v;
    }
    __syncwarp();
  }
}

}  // namespace bsidmap
