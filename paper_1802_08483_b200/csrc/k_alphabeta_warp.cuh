// k_alphabeta_warp.cuh -- a2/a3 for small trellises (M_tau <= 128): one warp per
// (frame, direction), SPT = ceil(M_tau / 32) states per lane, no block barrier.
//
//   alpha'_{i+1}(m) = sum_k alpha_i(m - k) Gamma_i(m - k, k)      (eqn:alpha_prenorm)
//   beta'_i(m')     = sum_k Gamma_i(m', k) beta_{i+1}(m' + k)     (eqn:beta)
// then division by the row sum (eqn:alpha_norm; "similar" for beta), FP64.
//
// The recursion is sequential in i and HBM-bound (it reads every Gamma_i block,
// M_n x Mtp FP32, once per direction).  Each warp streams its frame's Gamma_i
// blocks through a kStages-deep ring in shared memory with the TMA bulk-copy
// engine (cp.async.bulk ... mbarrier::complete_tx): lane 0 issues the copy of step
// i + kStages as soon as step i's block is consumed, so the copies overlap the
// FP64 arithmetic of the steps in between and no register holds prefetched data.
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace bsidmap {

#ifndef BSIDMAP_AB_WARP_THREADS
#define BSIDMAP_AB_WARP_THREADS 64
#endif
// 2 (frame, direction) tasks per CTA: finer-grained residency than 4 (C2: 9.38 -> 8.80 ms;
// 1 per CTA 15.8 ms; tools/exp_abw.sh)
constexpr int kAbWarpThreads = BSIDMAP_AB_WARP_THREADS;
// TMA ring depth per warp (C2: 2 stages 8.48 ms, 3: 8.35, 4: 8.80, 5: 8.87, 8: 14.1; tools/exp_abw2.sh)
#ifndef BSIDMAP_AB_STAGES
#define BSIDMAP_AB_STAGES 3
#endif
constexpr int kAbStages = BSIDMAP_AB_STAGES;

// shared memory per warp: row[MN + SPT*32 + MN] doubles (the state row with M_n zero entries on
// both sides and zeros at m >= M_tau) | ring[kStages][MN][Mtp] floats | bars[kStages]
__host__ __device__ __forceinline__ size_t ab_warp_row_bytes(int SPT, int MN) {
  return ((size_t)(SPT * 32 + 2 * MN) * 8 + 15) & ~(size_t)15;  // the TMA ring stays 16-byte aligned
}
__host__ __device__ __forceinline__ size_t ab_warp_smem(int SPT, int MN, int Mtp) {
  // rounded to 16 bytes: the next warp's TMA ring must stay 16-byte aligned
  return (ab_warp_row_bytes(SPT, MN) + (size_t)kAbStages * MN * Mtp * 4 + kAbStages * 8 + 15) & ~(size_t)15;
}

// The state row lives in shared memory with M_n zero entries on both sides and zeros for m >= M_tau,
// so the gathers need no bounds tests: beta reads row[m + k] (k = m_n^- + e) and Gamma column m, always
// inside [0, M_tau) for m < M_tau; alpha reads row[j] and Gamma column j = m - k, which is clamped into
// [0, M_tau) (its row factor is then 0).  Lanes with m >= M_tau compute a discarded value.
template <int SPT, int MN>
__global__ void __launch_bounds__(kAbWarpThreads) k_alpha_beta_warp(const DecodeParams p) {
  extern __shared__ __align__(128) unsigned char s_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Mt = p.Mt, Mtp = p.Mtp, N = p.N, lo = p.mn_lo;
  unsigned char* base = s_raw + (size_t)warp * ab_warp_smem(SPT, MN, Mtp);
  double* const rowx = reinterpret_cast<double*>(base);  // [MN + SPT*32 + MN]
  double* const row = rowx + MN;                         // row[m], m in [-MN, SPT*32 + MN)
  float* ring = reinterpret_cast<float*>(base + ab_warp_row_bytes(SPT, MN));
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + ab_warp_row_bytes(SPT, MN) + (size_t)kAbStages * MN * Mtp * 4);
  const long task = (long)blockIdx.x * (kAbWarpThreads / 32) + warp;
  const bool both = p.ab_dir < 0;  // (frame, direction) tasks, or one direction per frame
  if (task >= (both ? 2L : 1L) * p.F) return;  // warp-uniform
  const int f = (int)(both ? task >> 1 : task);
  const bool fwd = both ? (task & 1) == 0 : p.ab_dir == 0;
  const int r0 = p.ab_r0, r1 = p.ab_r1;  // steps of this launch (the whole recursion: 0, N)
  if (p.status[f] != kFrameOk) return;
  double* const arows = p.alpha + (size_t)f * (N + 1) * Mt;
  auto row_at = [&](int r) { return fwd ? arows + (size_t)r * Mt : beta_row(p, f, r); };
  const uint32_t blk_bytes = (uint32_t)(MN * Mtp * 4);
  auto gblock = [&](int step) { return gsum_block(p, f, fwd ? step : N - 1 - step); };

  if (lane == 0) {
    for (int s = 0; s < kAbStages; s++) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < kAbStages && r0 + s < r1; s++) {
      mbar_expect_tx(bars + s, blk_bytes);
      tma_bulk_g2s(ring + (size_t)s * MN * Mtp, gblock(r0 + s), blk_bytes, bars + s);
    }
  }
  for (int t = lane; t < SPT * 32 + 2 * MN; t += 32) rowx[t] = 0.0;
  __syncwarp();
  const int i0 = fwd ? r0 : N - r0;
#pragma unroll
  for (int s = 0; s < SPT; s++) {
    const int m = lane + 32 * s;
    if (m < Mt) {
      if (r0 == 0) {
        const double v = boundary_row(p, f, m, fwd);  // alpha_0 / beta_N
        row[m] = v;
        row_at(i0)[m] = v;
      } else {
        row[m] = row_at(i0)[m];  // resume from the stored, normalised row
      }
    }
  }
  __syncwarp();
  for (int step = r0; step < r1; step++) {
    const int t = step - r0;
    const int stage = t % kAbStages;
    mbar_wait(bars + stage, (uint32_t)(t / kAbStages) & 1u);
    const float* G = ring + (size_t)stage * MN * Mtp;  // Gamma_i [k][m'] in smem
    double acc[SPT];
    double part = 0.0;
#pragma unroll
    for (int s = 0; s < SPT; s++) {
      const int m = lane + 32 * s;
      double a0 = 0.0, a1 = 0.0;
      if (fwd) {  // alpha'(m) = sum_e alpha(j) Gamma(j, k), j = m - k, k = m_n^- + e
        const int j0 = m - lo;
#pragma unroll
        for (int e = 0; e < MN; e++) {
          const int j = j0 - e;
          const double g = (double)G[e * Mtp + min(max(j, 0), Mt - 1)];
          if (e & 1) a1 = fma(row[j], g, a1); else a0 = fma(row[j], g, a0);
        }
      } else {    // beta'(m) = sum_e Gamma(m, k) beta(m + k)
        const double* c0 = row + m + lo;
        const float* g0 = G + min(m, Mt - 1);
#pragma unroll
        for (int e = 0; e < MN; e++) {
          const double g = (double)g0[e * Mtp];
          if (e & 1) a1 = fma(g, c0[e], a1); else a0 = fma(g, c0[e], a0);
        }
      }
      acc[s] = m < Mt ? a0 + a1 : 0.0;
      part += acc[s];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    __syncwarp();  // every lane is done with this stage and with the old row
    if (lane == 0 && step + kAbStages < r1) {
      mbar_expect_tx(bars + stage, blk_bytes);
      tma_bulk_g2s(ring + (size_t)stage * MN * Mtp, gblock(step + kAbStages), blk_bytes, bars + stage);
    }
    if (!(part > 0.0)) {  // all-zero row: Y impossible under the limits (reading R14)
      if (lane == 0) p.status[f] = kFrameUnderflow;
      // drain the copies already issued for later steps before the warp's smem can be reused
      for (int u = t + 1; r0 + u < r1 && u <= t + kAbStages; u++)
        mbar_wait(bars + u % kAbStages, (uint32_t)(u / kAbStages) & 1u);
      return;
    }
    const double inv = 1.0 / part;
    const int r = fwd ? step + 1 : N - 1 - step;
    double* const out = row_at(r);
#pragma unroll
    for (int s = 0; s < SPT; s++) {
      const int m = lane + 32 * s;
      const double v = acc[s] * inv;
      row[m] = v;  // 0 for m >= M_tau
      if (m < Mt) out[m] = v;
    }
    __syncwarp();
  }
}

}  // namespace bsidmap
