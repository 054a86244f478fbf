// k_local_cta.cuh -- the paper's memory-reduced ("local storage") schedule for frames
// whose drift trellis does not fit one warp (M_tau > 64): one CTA of kLocalCtaThreads threads owns
// one frame for the whole pass; warps walk the frame's 32-state tiles.  gamma_i is computed inside
// the alpha pass and again inside the combined beta + L pass ("combining the computation of L with
// that of beta"); only the alpha rows are stored (8 (N+1) M_tau bytes per frame).
//
//   k_local_cta_fwd : for i = 0..N-1: Gamma_i(m', k) = sum_D P(D) G(m', k, D) for every window with
//                     alpha_i(m') != 0 (a window whose alpha is exactly 0 contributes exactly 0 to
//                     alpha_{i+1}: skipped) into a shared [M_n][M_tau] tile, then
//                     alpha_{i+1}(m) = sum_k alpha_i(m-k) Gamma_i(m-k, k) (eqn:alpha_prenorm),
//                     normalised (eqn:alpha_norm), row written to HBM (FP64).
//   k_local_cta_bwd : for i = N-1..0: t(m', D) = sum_k G(m', k, D) beta_{i+1}(m'+k) for every window,
//                     L_i(D) from sum_{m'} alpha_i(m') t(m', D) (eqn:L, written normalised) and
//                     beta_i(m') = sum_D P(D) t(m', D) (eqn:beta), normalised.
// Scalar lattice core (lattice.cuh); symbols visited in suffix-class order in the forward pass
// (last K rows once per class, as pass 1), the last row folded into the weights in the backward
// pass (as the APP pass).  Three block barriers per step.
#pragma once
#include "k_lattice_x2.cuh"

namespace bsidmap {

constexpr int kLocalCtaThreads = 256;
// frames (CTAs) per SM: 2 (128 registers per thread) measured faster for M_n <= 20 (C3: 268 vs
// 399 ms per 2048 frames), 1 for wider corridors (C4: 321 vs 339 ms) -- tools/exp_lcta.sh
#ifndef BSIDMAP_LOCAL_CTA_MINB
#define BSIDMAP_LOCAL_CTA_MINB (Core::Mn <= 20 ? 2 : 1)
#endif
constexpr int kLocalCtaWarps = kLocalCtaThreads / 32;

// fwd smem: s_res[M_n][256] floats | s_G[M_n][Mtp] floats | row[M_n + Mtp + M_n] doubles | part[32] doubles
__host__ __device__ __forceinline__ size_t local_cta_fwd_smem(int Mn, int Mtp) {
  return (size_t)Mn * kLocalCtaThreads * 4 + (size_t)Mn * Mtp * 4 + (size_t)(Mtp + 2 * Mn) * 8 + 32 * 8;
}
// bwd smem: stage[8][q][33] floats | Sd[q] doubles | beta rows 2 x [M_n + Mtp + M_n] doubles | part[2][32]
__host__ __device__ __forceinline__ size_t local_cta_bwd_smem(int Mn, int Mtp, int q) {
  return (size_t)kLocalCtaWarps * app_stage_floats(q) * 4 + (size_t)q * 8 + 2 * (size_t)(Mtp + 2 * Mn) * 8 +
         64 * 8;
}

// block-wide sum of one double per thread (all threads get the result); part: 32 doubles of smem
__device__ __forceinline__ double block_sum(double v, double* part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();  // part may still be read from a previous call
  if (lane == 0) part[warp] = v;
  __syncthreads();
  double c = lane < kLocalCtaWarps ? part[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  return c;
}

template <class Core, int K, bool kPri>
__global__ void __launch_bounds__(kLocalCtaThreads, BSIDMAP_LOCAL_CTA_MINB) k_local_cta_fwd(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  constexpr int NC = 1 << K;
  extern __shared__ __align__(128) unsigned char smem[];
  const int Mt = p.Mt, Mtp = p.Mtp, N = p.N, lo = p.mn_lo;
  float* s_res = reinterpret_cast<float*>(smem) + threadIdx.x;  // [MN][256], this thread's column
  float* s_G = reinterpret_cast<float*>(smem) + (size_t)MN * kLocalCtaThreads;  // Gamma_i [e][m']
  double* row = reinterpret_cast<double*>(s_G + (size_t)MN * Mtp) + MN;   // alpha_i, zero margins
  double* part = row + Mtp + MN;
  const int f = blockIdx.x;
  if (p.status[f] != kFrameOk) return;  // uniform over the CTA
  const int tid = threadIdx.x;
  double* rows_g = p.alpha + (size_t)f * (N + 1) * Mt;
  for (int t = tid; t < Mtp + 2 * MN; t += kLocalCtaThreads) row[t - MN] = 0.0;
  __syncthreads();
  for (int m = tid; m < Mt; m += kLocalCtaThreads) {
    const double v = boundary_row(p, f, m, true);  // alpha_0
    row[m] = v;
    rows_g[m] = v;
  }
  __syncthreads();
  const float sc = kPri ? 1.f : 1.f / p.q;
  for (int i = 0; i < N; i++) {
    const uint32_t* Ci = p.Cs[K - 2] + (size_t)i * p.q;
    const uint16_t* Di = p.Ds[K - 2] + (size_t)i * p.q;
    const int* cst = p.Cst[K - 2] + (size_t)i * (NC + 1);
    const float* pri = kPri ? p.priors + ((size_t)f * N + i) * p.q : nullptr;
    for (int m0 = (tid >> 5) * 32; m0 < Mt; m0 += kLocalCtaThreads) {  // warp tiles of 32 windows
      const int mi = m0 + (tid & 31);
      const LaneGeom G = geom_fm(p, i, f, mi, mi < Mt);
      const bool need = G.active && row[mi] != 0.0;  // alpha_i(m') = 0: Gamma_i(m', .) is not needed
      float acc[MN];
#pragma unroll
      for (int e = 0; e < MN; e++) acc[e] = 0.f;
      if (__any_sync(0xffffffffu, need)) {
        typename Core::Lane lane;
        Core::init(lane, need ? load_window(p, f, G.s, G.rho) : 0ull, p);
        bool first = true;
        int k = 0;
        XPrefetch xs(Ci, 0, p.q);
#pragma unroll 1
        for (int c = 0; c < NC; c++) {
          const int kend = cst[c + 1];
          if (k == kend) continue;
#pragma unroll
          for (int e = 0; e < MN; e++) acc[e] = 0.f;
          for (; k < kend; k++) {
            float fo[MN];
            Core::template run_prefix<K>(lane, xs.take(k), p, fo);
            if constexpr (kPri) {
              const float P = __ldg(pri + Di[k]);
#pragma unroll
              for (int e = 0; e < MN; e++) acc[e] = fmaf(P, fo[e], acc[e]);
            } else {
#pragma unroll
              for (int e = 0; e < MN; e++) acc[e] += fo[e];
            }
          }
          Core::template apply_last_rows<K>(lane, (uint32_t)c, p, acc);
#pragma unroll
          for (int e = 0; e < MN; e++) {
            if (!first) acc[e] += s_res[e * kLocalCtaThreads];
            s_res[e * kLocalCtaThreads] = acc[e];
          }
          first = false;
        }
      }
      if (mi < Mt) {
#pragma unroll
        for (int e = 0; e < MN; e++) s_G[e * Mtp + mi] = (need && out_valid(p, G, e)) ? sc * acc[e] : 0.f;
      }
    }
    __syncthreads();  // the Gamma_i tile is complete
    // alpha'_{i+1}(m) = sum_k alpha_i(m - k) Gamma_i(m - k, k): column j = m - lo - e (clamped where the
    // alpha factor is a zero margin); M_tau <= 4 x 256 (planner)
    double nv[4];
    double ps = 0.0;
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int m = tid + r * kLocalCtaThreads;
      double a0 = 0.0, a1 = 0.0;
      if (m < Mt) {
#pragma unroll
        for (int e = 0; e < MN; e++) {
          const int j = m - lo - e;
          const double t = row[j] * (double)s_G[e * Mtp + min(max(j, 0), Mt - 1)];
          if (e & 1) a1 += t; else a0 += t;
        }
      }
      nv[r] = a0 + a1;
      ps += nv[r];
    }
    const double c = block_sum(ps, part);  // also orders the tile reads before the row update
    if (!(c > 0.0)) {  // all-zero row (reading R14)
      if (tid == 0) p.status[f] = kFrameUnderflow;
      return;
    }
    const double inv = 1.0 / c;
    double* out = rows_g + (size_t)(i + 1) * Mt;
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int m = tid + r * kLocalCtaThreads;
      if (m < Mt) {
        row[m] = nv[r] * inv;  // eqn:alpha_norm
        out[m] = nv[r] * inv;
      }
    }
    __syncthreads();  // alpha_{i+1} complete before the next step reads it
  }
}

template <class Core, bool kPri>
__global__ void __launch_bounds__(kLocalCtaThreads, BSIDMAP_LOCAL_CTA_MINB) k_local_cta_bwd(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  extern __shared__ __align__(128) unsigned char smem[];
  const int Mt = p.Mt, Mtp = p.Mtp, N = p.N, lo = p.mn_lo;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* stg = reinterpret_cast<float*>(smem) + (size_t)warp * app_stage_floats(p.q);
  double* Sd = reinterpret_cast<double*>(reinterpret_cast<float*>(smem) + (size_t)kLocalCtaWarps * app_stage_floats(p.q));
  double* rowA = Sd + p.q + MN;  // beta rows with zero margins (ping-pong)
  double* rowB = rowA + Mtp + 2 * MN;
  double* part = rowB + Mtp + MN;
  const int f = blockIdx.x;
  float* Lf = p.L + (size_t)f * N * p.q;
  if (p.status[f] != kFrameOk) {  // failed frame: zero rows
    for (long k = tid; k < (long)N * p.q; k += kLocalCtaThreads) Lf[k] = 0.f;
    return;
  }
  const double* alpha_f = p.alpha + (size_t)f * (N + 1) * Mt;
  for (int t = tid; t < Mtp + 2 * MN; t += kLocalCtaThreads) {
    rowA[t - MN] = 0.0;
    rowB[t - MN] = 0.0;
  }
  __syncthreads();
  for (int m = tid; m < Mt; m += kLocalCtaThreads) rowA[m] = boundary_row(p, f, m, false);  // beta_N
  const int nb = p.n - 1;
  double* cur = rowA;  // beta_{i+1}
  double* nxt = rowB;  // beta_i
  for (int i = N - 1; i >= 0; i--) {
    __syncthreads();  // the previous step's readers of Sd and writers of cur are done
    for (int t = tid; t < p.q; t += kLocalCtaThreads) Sd[t] = 0.0;
    __syncthreads();  // Sd cleared, cur complete
    const uint32_t* Ci = p.C + (size_t)i * p.q;
    const float* pri = kPri ? p.priors + ((size_t)f * N + i) * p.q : nullptr;
    double bsum = 0.0;
    for (int m0 = warp * 32; m0 < Mt; m0 += kLocalCtaThreads) {  // warp tiles of 32 windows
      const int mi = m0 + lane;
      const LaneGeom G = geom_fm(p, i, f, mi, mi < Mt);
      // beta_{i+1}(m' + k) scaled by 2^-E (E: exponent of the corridor max) and w = alpha_i(m') 2^E
      float bt[MN];
      int hm = 0;
#pragma unroll
      for (int e = 0; e < MN; e++)
        if ((G.vmask >> e) & 1u) hm = max(hm, __double2hiint(cur[mi + lo + e]));
      const int E = hm > 0 ? (hm >> 20) - 1023 : 0;
      const double s = pow2d(-E);
#pragma unroll
      for (int e = 0; e < MN; e++) bt[e] = ((G.vmask >> e) & 1u) ? (float)(cur[mi + lo + e] * s) : 0.f;
      const double da = (G.active && hm > 0) ? alpha_f[(size_t)i * Mt + mi] * pow2d(E) : 0.0;
      const int Emax = __reduce_max_sync(0xffffffffu, da > 0.0 ? exp2_of(da) + 2048 : 0) - 2048;
      const float wa = (float)(da * pow2d(-Emax));
      const bool live = __any_sync(0xffffffffu, G.active && hm > 0);
      float bacc = 0.f;  // sum_D P(D) t(m', D)
      if (live) {
        typename Core::Lane lt;
        Core::init(lt, G.active ? load_window(p, f, G.s, G.rho) : 0ull, p);
        float w1[MN], w0[MN];  // the last lattice row folded into the weights (one table per x_n)
        Core::last_row_weights(lt, bt, w1, w0);
        XPrefetch xs(Ci, 0, p.q);
        for (int D = 0; D < p.q; D++) {
          const uint32_t x = xs.take(D);
          float fo[MN];
          Core::run_penultimate(lt, x, p, fo);
          float t0 = 0.f, t1 = 0.f;
          if ((x >> nb) & 1u) {
#pragma unroll
            for (int e = 0; e < MN; e += 2) {
              t0 = fmaf(fo[e], w1[e], t0);
              if (e + 1 < MN) t1 = fmaf(fo[e + 1], w1[e + 1], t1);
            }
          } else {
#pragma unroll
            for (int e = 0; e < MN; e += 2) {
              t0 = fmaf(fo[e], w0[e], t0);
              if (e + 1 < MN) t1 = fmaf(fo[e + 1], w0[e + 1], t1);
            }
          }
          const float t = t0 + t1;
          const float P = kPri ? __ldg(pri + D) : 1.f;
          bacc = fmaf(P, t, bacc);
          stg[D * 33 + lane] = wa * t;
        }
        __syncwarp();
        const double wsc = pow2d(Emax);
        for (int D = lane; D < p.q; D += 32) {  // this tile's share of S_i(D) = P(D) sum_m' alpha t
          float c = 0.f;
#pragma unroll 8
          for (int l = 0; l < 32; l++) c += stg[D * 33 + l];
          const float P = kPri ? __ldg(pri + D) : 1.f;
          if (c > 0.f) atomicAdd(Sd + D, (double)(c * P) * wsc);
        }
        __syncwarp();
      }
      // beta'_i(m') = 2^E sum_D P(D) t(m', D)  (eqn:beta)
      const double bv = (mi < Mt && G.active && hm > 0) ? (double)bacc * pow2d(E) : 0.0;
      if (mi < Mt) nxt[mi] = bv;
      bsum += bv;
    }
    const double c = block_sum(bsum, part);  // all tiles done: Sd and nxt complete
    // L_i(D) = S(D) / sum_D S(D)   (eqn:L; the literal 1/lambda_N in exact arithmetic, reading R2)
    double tot = 0.0;
    for (int D = 0; D < p.q; D++) tot += Sd[D];
    const bool ok = tot > 0.0 && c > 0.0;
    float* Lrow = Lf + (size_t)i * p.q;
    for (int D = tid; D < p.q; D += kLocalCtaThreads) Lrow[D] = ok ? (float)(Sd[D] / tot) : 0.f;
    if (!ok) {
      if (tid == 0) p.status[f] = kFrameUnderflow;
      return;
    }
    const double inv = 1.0 / c;  // eqn:beta normalisation
    for (int m = tid; m < Mt; m += kLocalCtaThreads) nxt[m] *= inv;
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
}

}  // namespace bsidmap

namespace bsidmap {
// kernel table of the CTA local schedule for one scalar spec core
template <class Core>
void local_cta_kernels(CoreKernels* k) {
  k->local_cta_fwd[0][0] = k_local_cta_fwd<Core, 2, false>;
  k->local_cta_fwd[0][1] = k_local_cta_fwd<Core, 2, true>;
  k->local_cta_fwd[1][0] = k_local_cta_fwd<Core, 3, false>;
  k->local_cta_fwd[1][1] = k_local_cta_fwd<Core, 3, true>;
  k->local_cta_bwd[0] = k_local_cta_bwd<Core, false>;
  k->local_cta_bwd[1] = k_local_cta_bwd<Core, true>;
}
}  // namespace bsidmap
