// k_app_live.cuh -- the APP pass (row a4, eqn:L / eqn:sigma, the second lattice pass of the
// memory-reduced variant) over the LIVE windows only.
//
//   S_i(D) = sum_{m' live} alpha_i(m') sum_k gamma_i(m', m'+k, D) beta_{i+1}(m'+k),
//   L_i(D) = P(D) S_i(D) / sum_D P(D) S_i(D)      (priors as in eqn:gamma)
//
// k_live (k_states.cu) marks, per APP row (f, i), the state range of the windows whose posterior
// mass alpha_i(m') beta_i(m') exceeds eps of the row's (reading R18).  Away from the posterior
// drift most windows are dead (C2: 24 of 62 states live, C3: 74 of 267, C4: 91 of 611, C5: 29 of
// 906 at eps = 2^-128), so the windows are packed instead of tiled: a warp owns G frames at one
// symbol index i and walks their live windows in rounds of 32 W (W windows per lane, every lane
// on the same C_i(D), so the lattice rows stay warp-uniform); each lane's per-symbol term is staged
// in shared memory and added, per frame, into FP64 sums S[G][q]; at the end the warp writes the G
// normalised L rows itself (no FP64 atomics, no finalize pass).
#pragma once
#include "k_lattice_x2.cuh"

namespace bsidmap {

constexpr int kLiveMaxG = 16;  // frames per warp (p.app_G <= kLiveMaxG)

// smem per warp of the pair kernel: weight tables [NT][M_n][32] f32x2 | S[G][q] double |
// stage [q][33] double | frame slot per lane [32] int
__host__ __device__ __forceinline__ size_t app_live_x2_warp_smem(int q, int Mn, int ks, int G) {
  const size_t b = (size_t)(2 << (ks - 1)) * Mn * 32 * 8 + (size_t)G * q * 8 + (size_t)q * 33 * 8 + 32 * 4;
  return (b + 15) & ~size_t(15);
}
// scalar kernel: weight tables of the whole CTA [4][M_n][128] float (KS = 2) first, then per warp
// S[G][q] double | scale per lane [32] double | stage [q][33] float | frame slot per lane [32] int
__host__ __device__ __forceinline__ size_t app_live_x1_warp_smem(int q, int G) {
  const size_t b = (size_t)G * q * 8 + 32 * 8 + (size_t)q * 33 * 4 + 32 * 4;
  return (b + 15) & ~size_t(15);
}
__host__ __device__ __forceinline__ size_t app_live_x1_cta_tables(int Mn, int ks) {
  return ks == 2 ? (size_t)4 * Mn * kLatticeThreads * 4 : 0;
}

// The warp's G frames at symbol index i: lane g < G holds (first live state, count) of frame f0 + g
// and its exclusive offset in the warp's window list; returns the list length.
struct LiveRows {
  int lo, cnt, ex, total;
};
__device__ __forceinline__ LiveRows live_rows(const DecodeParams& p, int f0, int i, int lane) {
  LiveRows r;
  int2 lv = make_int2(0, 0);
  if (lane < p.app_G && f0 + lane < p.F) lv = p.live[(size_t)(f0 + lane) * p.N + i];
  r.lo = lv.x;
  r.cnt = lv.y;
  int inc = r.cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  r.ex = inc - r.cnt;
  r.total = __shfl_sync(0xffffffffu, inc, 31);
  return r;
}
// frame slot g of list entry e (< total): the last frame whose exclusive offset is <= e (frames
// without live windows share their successor's offset and are passed over)
__device__ __forceinline__ int live_slot(const LiveRows& r, int G, int e) {
  int g = 0;
  for (int h = 1; h < G; h++)
    if (__shfl_sync(0xffffffffu, r.ex, h) <= e) g = h;
  return g;
}

// Per-frame FP64 sums of the staged per-lane terms: lanes of one frame are contiguous.  (A frame
// split over two rounds is summed as two partial sums: the FP64 association depends on the packing,
// far below the FP32 rounding of L -- tested bit-identical over G in test_live_app_independent_of_packing;
// a strictly sequential order measured 20 % slower on C2's APP.)
template <class T>
__device__ __forceinline__ void live_reduce(const DecodeParams& p, const T* stg, const double* sc, const int* sg,
                                            double* S, int lane) {
  for (int D = lane; D < p.q; D += 32) {
    double acc = 0.0;
    int cur = sg[0];
#pragma unroll 4
    for (int l = 0; l < 32; l++) {
      const int gl = sg[l];
      if (gl != cur) {
        if (cur >= 0) S[cur * p.q + D] += acc;
        acc = 0.0;
        cur = gl;
      }
      acc += sc ? (double)stg[D * 33 + l] * sc[l] : (double)stg[D * 33 + l];
    }
    if (cur >= 0) S[cur * p.q + D] += acc;
  }
}

// L_i(D) = P(D) S(D) / sum_D P(D) S(D) for the warp's G frames (FP64, FP32 output); a frame OK so far
// whose row sums to 0 is UNDERFLOW (reading R14).
__device__ __forceinline__ void live_write_rows(const DecodeParams& p, const double* S, int f0, int i, int lane) {
  for (int g = 0; g < p.app_G; g++) {
    const int f = f0 + g;
    if (f >= p.F) break;
    const float* pri = p.priors ? p.priors + ((size_t)f * p.N + i) * p.q : nullptr;
    double tot = 0.0;
    for (int D = lane; D < p.q; D += 32) tot += S[g * p.q + D] * (pri ? (double)__ldg(pri + D) : 1.0);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    const bool frame_ok = p.status[f] == kFrameOk;
    const bool ok = frame_ok && tot > 0.0;
    const double inv = ok ? 1.0 / tot : 0.0;
    float* Lrow = p.L + ((size_t)f * p.N + i) * p.q;
    for (int D = lane; D < p.q; D += 32)
      Lrow[D] = ok ? (float)(S[g * p.q + D] * (pri ? (double)__ldg(pri + D) : 1.0) * inv) : 0.f;
    if (frame_ok && !ok && lane == 0) p.status[f] = kFrameUnderflow;
  }
}

#ifndef BSIDMAP_LIVE_MINB
#define BSIDMAP_LIVE_MINB (Core::kMinBlocks > 2 ? 4 : 2)
#endif
// Pair core: two adjacent windows (m', m'+1) of one frame per lane; their terms are combined in
// FP64 (alpha beta weights of two windows may be far apart in scale).
template <class Core, int KP, int KS = 1>
__global__ void __launch_bounds__(kLatticeThreads, KS == 2 ? BSIDMAP_APP_MINB_KS2 : BSIDMAP_LIVE_MINB)
    k_app_live_x2(const DecodeParams p) {
  using f32x2 = typename Core::P2;
  constexpr int MN = Core::Mn;
  constexpr int NT = 2 << (KS - 1);  // weight tables per lane
  constexpr int RL = Core::NNr - KS;  // last lattice row run per symbol
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ws = smem + (size_t)warp * app_live_x2_warp_smem(p.q, MN, KS, p.app_G);
  f32x2* wt = reinterpret_cast<f32x2*>(ws) + lane;                       // [NT * MN][32]
  double* S = reinterpret_cast<double*>(ws + (size_t)NT * MN * 32 * 8);   // [G][q]
  double* stg = S + p.app_G * p.q;                                         // [q][33]
  int* sg = reinterpret_cast<int*>(stg + p.q * 33);                        // [32]
  const int i = blockIdx.y + p.i_base;
  const int f0 = (blockIdx.x * kX2Warps + warp) * p.app_G;
  if (f0 >= p.F) return;  // warp-uniform; no block barrier in this kernel
  const uint32_t* Ci = (KP > 0 ? p.Cp : p.C) + (size_t)i * p.q;
  const uint16_t* Di = p.Dp + (size_t)i * p.q;
  const LiveRows R = live_rows(p, f0, i, lane);
  for (int k = lane; k < p.app_G * p.q; k += 32) S[k] = 0.0;

  for (int r0 = 0; r0 < R.total; r0 += 64) {
    const int e = r0 + 2 * lane;
    const bool in = e < R.total;
    const int g = live_slot(R, p.app_G, e);  // every lane: the search shuffles
    const int lo = __shfl_sync(0xffffffffu, R.lo, g), ex = __shfl_sync(0xffffffffu, R.ex, g);
    const int f = f0 + g, mia = lo + (e - ex);
    const LaneGeom A = geom_fm(p, i, f, mia, in && mia < p.Mt);
    const LaneGeom B = geom_fm(p, i, f, mia + 1, in && mia + 1 < p.Mt);
    f32x2 bt[MN];
    double da, db;
    {
      float ba[MN], bb[MN];
      app_weights_pair<MN>(p, A, B, i, ba, bb, da, db);
#pragma unroll
      for (int u = 0; u < MN; u++) bt[u] = Core::pk(ba[u], bb[u]);
    }
    sg[lane] = in ? g : -1;  // the frame's lanes stay one segment (a window of weight 0 adds 0.0)
    if (__any_sync(0xffffffffu, da > 0.0 || db > 0.0)) {
      typename Core::Lane lane_t;
      Core::init(lane_t, A.active ? load_window(p, A.f, A.s, A.rho) : 0ull,
                 B.active ? load_window(p, B.f, B.s, B.rho) : 0ull, p);
      if constexpr (KS == 1) {
        Core::last_row_weights(lane_t, [&](int u) { return bt[u]; }, [&](int u) -> f32x2& { return wt[u * 32]; },
                               [&](int u) -> f32x2& { return wt[(MN + u) * 32]; });
      } else {
        f32x2 w1[MN], w0[MN], wi[MN];
        Core::last_row_weights(lane_t, [&](int u) { return bt[u]; }, [&](int u) -> f32x2& { return w1[u]; },
                               [&](int u) -> f32x2& { return w0[u]; });
        const f32x2 a2 = Core::pk(p.lc.a, p.lc.a);
        Core::template row_transpose<Core::NNr - 1>(w1, wi, lane_t.q1, a2);  // (x_{n-1}, x_n) = (1, 1)
#pragma unroll
        for (int u = 0; u < MN; u++) wt[u * 32] = wi[u];
        Core::template row_transpose<Core::NNr - 1>(w1, wi, lane_t.q0, a2);  // (0, 1)
#pragma unroll
        for (int u = 0; u < MN; u++) wt[(MN + u) * 32] = wi[u];
        Core::template row_transpose<Core::NNr - 1>(w0, wi, lane_t.q1, a2);  // (1, 0)
#pragma unroll
        for (int u = 0; u < MN; u++) wt[(2 * MN + u) * 32] = wi[u];
        Core::template row_transpose<Core::NNr - 1>(w0, wi, lane_t.q0, a2);  // (0, 0)
#pragma unroll
        for (int u = 0; u < MN; u++) wt[(3 * MN + u) * 32] = wi[u];
      }
      const int nb = p.n - 1;
      f32x2 fh[MN];  // rows 1..KP of the current prefix
      XPrefetch xs(Ci, 0, p.q);
      uint32_t xprev = 0u;
      for (int k = 0; k < p.q; k++) {
        const uint32_t x = xs.take(k);
        f32x2 fo[MN];
        // t(m', D) = sum_k G_n(m', k, D) bt(m', k) = sum_e G_{n-KS}[e] w[e]  (two chains)
        const f32x2* W = KS == 1 ? wt + (((x >> nb) & 1u) ? 0 : MN * 32)
                                 : wt + (size_t)((((x >> nb) & 1u) ? 0 : 2) + (((x >> (nb - 1)) & 1u) ? 0 : 1)) * MN * 32;
        f32x2 t0 = Core::f2z(), t1 = Core::f2z();
        auto dot = [&](const f32x2 (&gg)[MN]) {
#pragma unroll
          for (int u = 0; u < MN; u += 2) {
            t0 = ffma2(gg[u], W[u * 32], t0);
            if (u + 1 < MN) t1 = ffma2(gg[u + 1], W[(u + 1) * 32], t1);
          }
        };
        if constexpr (KP > 0) {
          if (k == 0 || ((x ^ xprev) & ((1u << KP) - 1u)) != 0u)
            Core::template run_head<KP, BSIDMAP_APP_GROUP>(lane_t, x, p, fh);
          xprev = x;
          Core::template run_tail_from_then<KP, RL, BSIDMAP_APP_GROUP>(lane_t, x, p, fh, fo, dot);
        } else {
          Core::template run_to_then<RL, BSIDMAP_APP_GROUP>(lane_t, x, p, fo, dot);
        }
        const int D = KP > 0 ? (int)Di[k] : k;
        stg[D * 33 + lane] =
            (da > 0.0 || db > 0.0) ? fma(da, (double)(lo_of(t0) + lo_of(t1)), db * (double)(hi_of(t0) + hi_of(t1))) : 0.0;
      }
    } else {
      for (int D = 0; D < p.q; D++) stg[D * 33 + lane] = 0.0;
    }
    __syncwarp();
    live_reduce<double>(p, stg, nullptr, sg, S, lane);
    __syncwarp();
  }
  live_write_rows(p, S, f0, i, lane);
}

#ifndef BSIDMAP_LIVE1_MINB
#define BSIDMAP_LIVE1_MINB 3
#endif
// Scalar core: one window per lane; the lane's alpha beta weight is scaled into [1, 2) by its own
// power of two (kept beside the staged FP32 term and applied in the FP64 sum).
template <class Core, int KP, int KS = 1>
__global__ void __launch_bounds__(kLatticeThreads, BSIDMAP_LIVE1_MINB) k_app_live_x1(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  constexpr int RL = Core::NNr - KS;  // last lattice row run per symbol
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* s_w = reinterpret_cast<float*>(smem) + threadIdx.x;  // KS = 2: [4][MN][128]
  unsigned char* ws = smem + app_live_x1_cta_tables(MN, KS) + (size_t)warp * app_live_x1_warp_smem(p.q, p.app_G);
  double* S = reinterpret_cast<double*>(ws);     // [G][q]
  double* sc = S + p.app_G * p.q;                // [32]
  float* stg = reinterpret_cast<float*>(sc + 32);  // [q][33]
  int* sg = reinterpret_cast<int*>(stg + p.q * 33);  // [32]
  const int i = blockIdx.y + p.i_base;
  const int f0 = (blockIdx.x * kX2Warps + warp) * p.app_G;
  if (f0 >= p.F) return;  // warp-uniform; no block barrier in this kernel
  const uint32_t* Ci = (KP > 0 ? p.Cp : p.C) + (size_t)i * p.q;
  const uint16_t* Di = p.Dp + (size_t)i * p.q;
  const LiveRows R = live_rows(p, f0, i, lane);
  for (int k = lane; k < p.app_G * p.q; k += 32) S[k] = 0.0;

  for (int r0 = 0; r0 < R.total; r0 += 32) {
    const int e = r0 + lane;
    const bool in = e < R.total;
    const int g = live_slot(R, p.app_G, e);  // every lane: the search shuffles
    const int lo = __shfl_sync(0xffffffffu, R.lo, g), ex = __shfl_sync(0xffffffffu, R.ex, g);
    const int f = f0 + g, mi = lo + (e - ex);
    const LaneGeom A = geom_fm(p, i, f, mi, in && mi < p.Mt);
    float bt[MN];
    const double da = app_weights_p2<MN>(p, A, i, bt);
    const int E = da > 0.0 ? exp2_of(da) : 0;
    const float wa = (float)(da * pow2d(-E));
    sg[lane] = in ? g : -1;  // the frame's lanes stay one segment (a window of weight 0 adds 0.0)
    sc[lane] = pow2d(E);
    if (__any_sync(0xffffffffu, da > 0.0)) {
      typename Core::Lane lane_t;
      Core::init(lane_t, A.active ? load_window(p, A.f, A.s, A.rho) : 0ull, p);
      float w1[MN], w0[MN];  // last lattice row folded into the weights (one table per x_n)
      Core::last_row_weights(lane_t, bt, w1, w0);
      if constexpr (KS == 2) {  // table c = 2 [x_n = 0] + [x_{n-1} = 0], entry e at s_w[(c MN + e) 128]
        float wi[MN];
        Core::template row_transpose<Core::NNr - 1>(w1, wi, lane_t.q1, p.lc.a);
#pragma unroll
        for (int u = 0; u < MN; u++) s_w[u * kLatticeThreads] = wi[u];
        Core::template row_transpose<Core::NNr - 1>(w1, wi, lane_t.q0, p.lc.a);
#pragma unroll
        for (int u = 0; u < MN; u++) s_w[(MN + u) * kLatticeThreads] = wi[u];
        Core::template row_transpose<Core::NNr - 1>(w0, wi, lane_t.q1, p.lc.a);
#pragma unroll
        for (int u = 0; u < MN; u++) s_w[(2 * MN + u) * kLatticeThreads] = wi[u];
        Core::template row_transpose<Core::NNr - 1>(w0, wi, lane_t.q0, p.lc.a);
#pragma unroll
        for (int u = 0; u < MN; u++) s_w[(3 * MN + u) * kLatticeThreads] = wi[u];
      }
      const int nb = p.n - 1;
      float fh[MN];  // rows 1..KP of the current prefix
      XPrefetch xs(Ci, 0, p.q);
      uint32_t xprev = 0u;
      for (int k = 0; k < p.q; k++) {
        const uint32_t x = xs.take(k);
        const int D = KP > 0 ? (int)Di[k] : k;
        float fo[MN];
        float t0 = 0.f, t1 = 0.f;
        const float* W = s_w + (size_t)((((x >> nb) & 1u) ? 0 : 2) + (((x >> (nb - 1)) & 1u) ? 0 : 1)) * MN * kLatticeThreads;
        auto dot = [&](const float (&gg)[MN]) {
          if constexpr (KS == 2) {
#pragma unroll
            for (int u = 0; u < MN; u += 2) {
              t0 = fmaf(gg[u], W[u * kLatticeThreads], t0);
              if (u + 1 < MN) t1 = fmaf(gg[u + 1], W[(u + 1) * kLatticeThreads], t1);
            }
          }
        };
        if constexpr (KP > 0) {
          if (k == 0 || ((x ^ xprev) & ((1u << KP) - 1u)) != 0u) Core::template run_head<KP>(lane_t, x, p, fh);
          xprev = x;
          Core::template run_tail_from<KP, RL, KS == 2>(lane_t, x, p, fh, fo, dot);
        } else {
          if constexpr (KS == 2) Core::template run_to_then<RL>(lane_t, x, p, fo, dot);
          else Core::template run_to<RL>(lane_t, x, p, fo);
        }
        if constexpr (KS == 1) {
          if ((x >> nb) & 1u) {
#pragma unroll
            for (int u = 0; u < MN; u += 2) {
              t0 = fmaf(fo[u], w1[u], t0);
              if (u + 1 < MN) t1 = fmaf(fo[u + 1], w1[u + 1], t1);
            }
          } else {
#pragma unroll
            for (int u = 0; u < MN; u += 2) {
              t0 = fmaf(fo[u], w0[u], t0);
              if (u + 1 < MN) t1 = fmaf(fo[u + 1], w0[u + 1], t1);
            }
          }
        }
        stg[D * 33 + lane] = da > 0.0 ? wa * (t0 + t1) : 0.f;
      }
    } else {
      for (int D = 0; D < p.q; D++) stg[D * 33 + lane] = 0.f;
    }
    __syncwarp();
    live_reduce<float>(p, stg, sc, sg, S, lane);
    __syncwarp();
  }
  live_write_rows(p, S, f0, i, lane);
}

}  // namespace bsidmap
