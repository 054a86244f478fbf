// k_lattice_x4.cuh -- APP pass (row a4, the second lattice pass of the memory-reduced
// variant) on the four-window core SpecCoreX4.
//
// Geometry: a HALF-warp owns a tile of 64 consecutive start drifts m' of one frame at one
// symbol index i (lane t of the half: m' slots 4t .. 4t+3), so a warp covers two tiles (two
// frames when M_tau <= 64) and a CTA of 4 warps eight.  Per symbol D the lane runs the
// lattice rows 1..n-1 of its four windows (two interleaved FFMA2 chains, SpecCoreX4), folds
// the last row into beta weights kept in shared memory, and stages
//   c(lane, D) = sum_{k<4} w_k t_k(D),  t_k(D) = sum_e G_{n-1,k}[e] w_{x_n,k}[e]
// (eqn:L / eqn:sigma restated per window: w_k = alpha_i(m'_k) scaled, t_k = sum_m gamma beta).
// The half-warp sums give S_i(D) of its tile; with one tile per frame the half writes
// L_i(D) = P(D) S(D) / sum_D P(D) S(D) directly, else FP64 atomics into Lacc (k_finalize).
#pragma once
#include "k_lattice_x2.cuh"
#include "lattice_x4.cuh"

namespace bsidmap {

__host__ __device__ __forceinline__ size_t app_x4_smem(int q, int Mn) {
  return (size_t)kX2Warps * 4 * Mn * 32 * 8 + (size_t)q * 4 + (size_t)kX2Warps * (app_stage_floats(q) + 2 * q) * 4;
}

#ifndef BSIDMAP_APP4_MINB
#define BSIDMAP_APP4_MINB 3
#endif

template <class Core>
__global__ void __launch_bounds__(kLatticeThreads, BSIDMAP_APP4_MINB) k_app_x4(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  extern __shared__ __align__(128) unsigned char smem[];
  f32x2* s_w = reinterpret_cast<f32x2*>(smem);  // [warp][A1, A0, B1, B0][MN][32]
  uint32_t* s_C = reinterpret_cast<uint32_t*>(s_w + kX2Warps * 4 * MN * 32);
  float* s_S = reinterpret_cast<float*>(s_C + p.q);  // [warp][2][q]
  float* s_stage = s_S + kX2Warps * 2 * p.q;        // [warp][q][33]
  const int i = blockIdx.y + p.i_base;
  for (int t = threadIdx.x; t < p.q; t += blockDim.x) s_C[t] = p.C[(size_t)i * p.q + t];
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane >> 4, t = lane & 15;
  const int T = tiles_per_frame(p.Mt);
  const long ht0 = ((long)blockIdx.x * kX2Warps + warp) * 2;  // the warp's first half-tile
  if (ht0 / T >= p.F) return;                                  // warp-uniform; no block barrier follows
  const long ht = ht0 + h;
  const int f = (int)(ht / T);
  const bool fin = f < p.F;
  const int mi0 = (int)(ht % T) * kTileSlots + 4 * t;
  LaneGeom G[4];
#pragma unroll
  for (int k = 0; k < 4; k++) G[k] = geom_fm(p, i, f, mi0 + k, fin && mi0 + k < p.Mt);
  const bool frame_ok = fin && p.status[f] == kFrameOk;

  // received bits from s0 = n i + m'_0 (bits before the frame start read as 0: those windows are inactive)
  const int s0 = G[0].s;
  const int rho = fin ? p.rho[f] : 0;
  uint64_t win = 0ull;
  if (G[0].active || G[1].active || G[2].active || G[3].active)
    win = s0 >= 0 ? load_window(p, f, s0, rho) : (load_window(p, f, 0, rho) << (-s0));
  typename Core::Lane lt;
  Core::init(lt, win, p);

  // beta_{i+1}(m'_k + m_n^- + e), e < M_n, for the four windows: one corridor of M_n + 3 states
  f32x2* wt = s_w + (size_t)warp * 4 * MN * 32 + lane;  // table c, entry e at wt[(c * MN + e) * 32]
  double d[4];
  {
    double bv[MN + 3];
    const double* brow = p.beta + ((size_t)(fin ? f : 0) * (p.N + 1) + (i + 1)) * p.Mt;
#pragma unroll
    for (int u = 0; u < MN + 3; u++) bv[u] = __ldg(brow + min(max(mi0 + p.mn_lo + u, 0), p.Mt - 1));
    float bt[4][MN];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      double bm = 0.0;
#pragma unroll
      for (int e = 0; e < MN; e++) bm = fmax(bm, ((G[k].vmask >> e) & 1u) ? bv[k + e] : 0.0);
      const int E = bm > 0.0 ? exp2_of(bm) : 0;
      const double sc = pow2d(-E);
#pragma unroll
      for (int e = 0; e < MN; e++) bt[k][e] = ((G[k].vmask >> e) & 1u) ? (float)(bv[k + e] * sc) : 0.f;
      d[k] = (G[k].active && bm > 0.0) ? p.alpha[((size_t)f * (p.N + 1) + i) * p.Mt + G[k].mi] * pow2d(E) : 0.0;
    }
    Core::template last_row_weights<false>(
        lt, [&](int e) { return pk(bt[0][e], bt[1][e]); }, [&](int e) -> f32x2& { return wt[e * 32]; },
        [&](int e) -> f32x2& { return wt[(MN + e) * 32]; });
    Core::template last_row_weights<true>(
        lt, [&](int e) { return pk(bt[2][e], bt[3][e]); }, [&](int e) -> f32x2& { return wt[(2 * MN + e) * 32]; },
        [&](int e) -> f32x2& { return wt[(3 * MN + e) * 32]; });
  }
  // common power-of-two scale of the half-tile's weights
  int Emax;
  float w[4];
  {
    const double dm = fmax(fmax(d[0], d[1]), fmax(d[2], d[3]));
    int ex = dm > 0.0 ? exp2_of(dm) + 2048 : 0;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) ex = max(ex, __shfl_xor_sync(0xffffffffu, ex, o));
    Emax = ex - 2048;
    const double sc = pow2d(-Emax);
#pragma unroll
    for (int k = 0; k < 4; k++) w[k] = (float)(d[k] * sc);
  }
  const bool live = __any_sync(0xffffffffu, w[0] > 0.f || w[1] > 0.f || w[2] > 0.f || w[3] > 0.f);
  float* stg = s_stage + (size_t)warp * app_stage_floats(p.q);
  float* S = s_S + warp * 2 * p.q;
  const int nb = p.n - 1;
  if (live) {
    __syncwarp();
    for (int D = 0; D < p.q; D++) {
      const uint32_t x = s_C[D];
      f32x2 fa[MN], fb[MN];
      Core::run_penultimate(lt, x, p, fa, fb);
      const int c1 = ((x >> nb) & 1u) ? 0 : MN;  // table A1 / A0 (B: + 2 MN)
      const f32x2* WA = wt + c1 * 32;
      const f32x2* WB = wt + (2 * MN + c1) * 32;
      f32x2 ta0 = 0ull, ta1 = 0ull, tb0 = 0ull, tb1 = 0ull;
#pragma unroll
      for (int e = 0; e < MN; e += 2) {
        ta0 = ffma2(fa[e], WA[e * 32], ta0);
        tb0 = ffma2(fb[e], WB[e * 32], tb0);
        if (e + 1 < MN) {
          ta1 = ffma2(fa[e + 1], WA[(e + 1) * 32], ta1);
          tb1 = ffma2(fb[e + 1], WB[(e + 1) * 32], tb1);
        }
      }
      const f32x2 ta = fadd2(ta0, ta1), tb = fadd2(tb0, tb1);
      stg[D * 33 + lane] = fmaf(w[0], lo_of(ta), fmaf(w[1], hi_of(ta), fmaf(w[2], lo_of(tb), w[3] * hi_of(tb))));
    }
    __syncwarp();
    // S[hh][D] = P_f(D) sum over the half's 16 lanes
    for (int idx = lane; idx < 2 * p.q; idx += 32) {
      const int hh = idx >= p.q ? 1 : 0, D = idx - hh * p.q;
      const int fh = (int)((ht0 + hh) / T);
      float c = 0.f;
#pragma unroll
      for (int l = 0; l < 16; l++) c += stg[D * 33 + hh * 16 + l];
      const float* pri = (p.priors && fh < p.F) ? p.priors + ((size_t)fh * p.N + i) * p.q : nullptr;
      S[idx] = pri ? c * __ldg(pri + D) : c;
    }
  }
  __syncwarp();
  float* Sh = S + h * p.q;
  if (T == 1) {
    float tot = 0.f;
    if (live)
      for (int D = t; D < p.q; D += 16) tot += Sh[D];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (fin) {
      const bool ok = frame_ok && live && tot > 0.f;
      const float inv = ok ? 1.f / tot : 0.f;
      float* Lrow = p.L + ((size_t)f * p.N + i) * p.q;
      for (int D = t; D < p.q; D += 16) Lrow[D] = ok ? Sh[D] * inv : 0.f;
      if (frame_ok && !ok && t == 0) p.status[f] = kFrameUnderflow;
    }
  } else if (live && fin) {
    const double sc = pow2d(Emax);
    double* acc = p.Lacc + ((size_t)f * p.N + i) * p.q;
    for (int D = t; D < p.q; D += 16) {
      const float v = Sh[D];
      if (v > 0.f) atomicAdd(acc + D, (double)v * sc);
    }
  }
}

}  // namespace bsidmap

namespace bsidmap {
// The four-window APP instance of a spec shape, or nullptr where its registers would not fit
// three CTAs per SM (Q-dot table 4(J + 2) + two corridors 4 M_n registers).
template <int NN, int LO, int MN>
constexpr void (*app_x4_kernel())(const DecodeParams) {
  if constexpr (MN <= 16 && NN + LO + MN - 1 <= 20)
    return k_app_x4<SpecCoreX4<NN, LO, MN>>;
  else
    return nullptr;
}
}  // namespace bsidmap
