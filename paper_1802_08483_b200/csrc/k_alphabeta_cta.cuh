// k_alphabeta_cta.cuh -- rows a2/a3: the alpha and beta recursions for large M_tau, one CTA per
// (frame, direction), persistent over the N steps (eqn:alpha, eqn:beta, eqn:alpha_norm, P:145-154,
// P:257-271; FP64 states).
//
//   alpha'_{i+1}(m) = sum_k alpha_i(m - k) Gamma_i(m - k, k),   alpha_{i+1} = alpha' / sum_m alpha'
//   beta'_i(m')     = sum_k Gamma_i(m', k) beta_{i+1}(m' + k),  beta_i = beta' / sum beta'
//
// Gamma_i blocks (M_n x Mtp FP32, contiguous) stream through a `stages`-deep shared-memory ring by
// TMA bulk copies (one thread issues, an mbarrier per stage).  ONE block barrier per step: the row
// is kept unnormalised (R_{i+1} = (1/c_i) sum_k R_i Gamma_i with c_i from the previous step's
// per-warp partial sums) and rows are ping-ponged.  The two state rows carry M_n zero entries on
// both sides (and zeros in [M_tau, Mtp)), so the beta gather needs no bounds test and the alpha
// gather only for the M_n edge states at either end, whose Gamma column is clamped (the state
// factor is then 0).  MNT = compile-time M_n (spec shapes: fully unrolled gather) or 0 (runtime).
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace bsidmap {

// ring[stages][M_n][Mtp] floats | R[2][M_n + Mtp + M_n] doubles | part[2][32] doubles | bars[stages]
__host__ __device__ __forceinline__ size_t ab_cta_smem(int Mn, int Mtp, int stages) {
  return (size_t)stages * Mn * Mtp * 4 + 2 * (size_t)(Mtp + 2 * Mn) * 8 + 2 * 32 * 8 + (size_t)stages * 8;
}

template <int MNT, bool kRing = true>
__global__ void __launch_bounds__(1024) k_alpha_beta_cta(const DecodeParams p, int stages) {
  if constexpr (!kRing) stages = 0;
  extern __shared__ __align__(128) unsigned char smem[];
  const int Mt = p.Mt, Mtp = p.Mtp, N = p.N, lo = p.mn_lo;
  const int Mn = MNT > 0 ? MNT : p.Mn;
  const int RW = Mtp + 2 * Mn;  // row stride with margins
  float* ring = reinterpret_cast<float*>(smem);
  double* Rb = reinterpret_cast<double*>(smem + (size_t)stages * Mn * Mtp * 4);
  double* part = Rb + 2 * RW;
  uint64_t* bars = reinterpret_cast<uint64_t*>(part + 64);
  const int f = blockIdx.x;
  const bool fwd = p.ab_dir < 0 ? blockIdx.y == 0 : p.ab_dir == 0;
  const int r0 = p.ab_r0, r1 = p.ab_r1;  // steps of this launch (the whole recursion: 0, N)
  if (p.status[f] != kFrameOk) return;  // uniform over the CTA
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, lane = tid & 31, nw = (nt + 31) >> 5;
  double* const arows = p.alpha + (size_t)f * (N + 1) * Mt;
  auto row_at = [&](int r) { return fwd ? arows + (size_t)r * Mt : beta_row(p, f, r); };
  const uint32_t blk = (uint32_t)(Mn * Mtp * 4);
  auto gblock = [&](int step) { return gsum_block(p, f, fwd ? step : N - 1 - step); };
  // kRing = false: a Gamma_i block larger than shared memory (wide trellises, e.g. C4's channel at
  // N = 1e5: M_n x M_tau x 4 > 227 KB) -- the CTA reads it straight from global memory (L2)
  if (kRing && tid == 0) {
    for (int s = 0; s < stages; s++) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < stages && r0 + s < r1; s++) {
      mbar_expect_tx(bars + s, blk);
      tma_bulk_g2s(ring + (size_t)s * Mn * Mtp, gblock(r0 + s), blk, bars + s);
    }
  }
  for (int t = tid; t < 2 * RW; t += nt) Rb[t] = 0.0;
  __syncthreads();
  const int i0 = fwd ? r0 : N - r0;
  for (int m = tid; m < Mt; m += nt) {
    if (r0 == 0) {
      const double v = boundary_row(p, f, m, fwd);  // alpha_0 / beta_N
      Rb[Mn + m] = v;
      row_at(i0)[m] = v;
    } else {
      Rb[Mn + m] = row_at(i0)[m];  // resume from the stored, normalised row
    }
  }
  __syncthreads();
  // alpha gather of state m reads Gamma column j = m - lo - e, e < M_n: all inside [0, M_tau)
  // for m in [m_lo_in, m_hi_in]
  const int m_lo_in = lo + Mn - 1, m_hi_in = Mt - 1 + lo;
  double inv_c = 1.0;  // scale of the current row (any constant: every row is normalised by its sum)
  for (int step = r0; step < r1; step++) {
    const int ts = step - r0;
    const int stage = kRing ? ts % stages : 0;
    if constexpr (kRing) mbar_wait(bars + stage, (uint32_t)(ts / stages) & 1u);
    const float* G = kRing ? ring + (size_t)stage * Mn * Mtp : gblock(step);
    const double* cur = Rb + (ts & 1) * RW + Mn;
    double* nxt = Rb + ((ts + 1) & 1) * RW + Mn;
    double ps = 0.0;
    for (int m = tid; m < Mt; m += nt) {
      double a0 = 0.0, a1 = 0.0;
      if (fwd) {
        const int j0 = m - lo;  // column of e = 0; column of e is j0 - e
        if (m >= m_lo_in && m <= m_hi_in) {
#pragma unroll
          for (int e = 0; e < (MNT > 0 ? MNT : kMaxMn); e++) {
            if (MNT == 0 && e >= Mn) break;
            const double t = cur[j0 - e] * (double)G[e * Mtp + j0 - e];
            if (e & 1) a1 += t; else a0 += t;
          }
        } else {
          for (int e = 0; e < Mn; e++) {
            const int j = j0 - e;
            const double t = cur[j] * (double)G[e * Mtp + min(max(j, 0), Mt - 1)];
            if (e & 1) a1 += t; else a0 += t;
          }
        }
      } else {
        const double* c0 = cur + m + lo;  // beta_{i+1}(m + k), k = lo + e (zero margins)
#pragma unroll
        for (int e = 0; e < (MNT > 0 ? MNT : kMaxMn); e++) {
          if (MNT == 0 && e >= Mn) break;
          const double t = (double)G[e * Mtp + m] * c0[e];
          if (e & 1) a1 += t; else a0 += t;
        }
      }
      const double v = (a0 + a1) * inv_c;
      nxt[m] = v;
      ps += v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
    double* pp = part + ((ts + 1) & 1) * 32;
    if (lane == 0) pp[warp] = ps;
    __syncthreads();  // nxt and the partials are complete; the ring stage is consumed
    if (kRing && tid == 0 && step + stages < r1) {
      mbar_expect_tx(bars + stage, blk);
      tma_bulk_g2s(ring + (size_t)stage * Mn * Mtp, gblock(step + stages), blk, bars + stage);
    }
    double c = lane < nw ? pp[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (!(c > 0.0)) {  // all-zero row: Y impossible under the limits (reading R14)
      if (tid == 0) {
        p.status[f] = kFrameUnderflow;
        for (int u = ts + 1; kRing && r0 + u < r1 && u <= ts + stages; u++)  // drain issued copies
          mbar_wait(bars + u % stages, (uint32_t)(u / stages) & 1u);
      }
      return;
    }
    inv_c = 1.0 / c;
    const int r = fwd ? step + 1 : N - 1 - step;
    double* const out = row_at(r);
    for (int m = tid; m < Mt; m += nt) out[m] = nxt[m] * inv_c;  // eqn:alpha_norm
  }
}

}  // namespace bsidmap
