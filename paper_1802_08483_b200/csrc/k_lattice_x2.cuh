// k_lattice_x2.cuh -- lattice passes on the packed-pair core (SpecCoreX2).
//
// Geometry: frame-aligned warp tiles.  A tile is 64 consecutive start drifts
// m' of ONE frame at one symbol index i (blockIdx.y); lane t owns slots 2t and
// 2t+1.  A frame of M_tau states spans T = ceil(M_tau / 64) tiles; a CTA is 4
// tiles.  Because a warp never mixes frames, the symbol priors P(D_i = D) are
// warp-uniform and the APP sum over m' is a plain warp reduction.
//
//   k_gamma_sum_x2 : a1 -- Gamma_i(m', k) = sum_D P(D) G_n(m', k, D)  (eqn:gamma
//                    folded over D), and every gamma in the stored variant
//                    (flat geometry: two windows 128 apart per lane).
//   k_app_x2       : a4 -- second lattice pass (gamma recomputed):
//                    S_i(D) = sum_{m'} alpha_i(m') sum_k gamma_i(m', m'+k, D) beta_{i+1}(m'+k)
//                    (eqn:L/eqn:sigma).  With T = 1 the warp holds the whole sum and
//                    writes L_i(D) = S_i(D) / sum_D S_i(D) directly; with T > 1 the
//                    warps add FP64 partials into Lacc (k_finalize normalises).
#pragma once
#include "k_lattice.cuh"

namespace bsidmap {

constexpr int kTileSlots = 64;

// Symbol-loop codeword prefetch: x of iteration k + 1 is read from shared memory during
// iteration k, so the warp-uniform row branches of the next lattice do not wait on it.
struct XPrefetch {
  const uint32_t* s;
  int last;
  uint32_t nxt;
  __device__ __forceinline__ XPrefetch(const uint32_t* s_C, int k0, int q) : s(s_C), last(q - 1), nxt(s_C[k0]) {}
  __device__ __forceinline__ uint32_t take(int k) {
    const uint32_t x = nxt;
    nxt = s[min(k + 1, last)];
    return x;
  }
};
constexpr int kX2Warps = kLatticeThreads / 32;

__host__ __device__ __forceinline__ int tiles_per_frame(int Mt) { return (Mt + kTileSlots - 1) / kTileSlots; }

// Window geometry of frame f, state index mi at symbol index i.
__device__ __forceinline__ LaneGeom geom_fm(const DecodeParams& p, int i, int f, int mi, bool in) {
  LaneGeom G;
  G.in = in;
  G.f = in ? f : 0;
  G.mi = in ? mi : 0;
  G.mp = p.mt_lo + G.mi;
  G.s = p.n * i + G.mp;
  G.rho = in ? p.rho[G.f] : 0;
  G.active = in && p.status[G.f] == kFrameOk && G.s >= 0 && G.s <= G.rho;
  G.vmask = valid_mask(p, G);
  return G;
}

// 2^k as a double, k in [-1022, 1023] (exact; no division on the hot path)
__device__ __forceinline__ double pow2d(int k) {
  k = max(-1022, min(1023, k));
  return __hiloint2double((k + 1023) << 20, 0);
}
__device__ __forceinline__ int exp2_of(double x) {  // floor(log2 x) for normal x > 0
  return ((__double2hiint(x) >> 20) & 0x7ff) - 1023;
}

// Pass 1 uses flat geometry: lane t of a CTA owns windows g0 + t and g0 + t + 128
// (g = f M_tau + m' index, g0 = 256 blockIdx.x) -- no frame alignment needed here.
#ifndef BSIDMAP_L1_MINB
#define BSIDMAP_L1_MINB Core::kMinBlocks
#endif
// the class-ordered pass 1 at one more CTA/SM where 3 fit (128 registers, ~140 B of spills outside
// the row loop; tools/exp_minb.sh: C2 pass 1 52.98 -> 50.79 ms, C1 shape 0.205 -> 0.192 ms)
// and at 3 (168 registers, ~100 B of spills) for the 2-CTA shapes with M_n <= BSIDMAP_SCALAR_MN_MAX
// (whose APP runs on the scalar core): C3 pass 1 67.7 -> 62.2 ms, C5 226.1 -> 199.7 ms against the
// scalar class kernel; C4 (M_n = 26) stays at 2 (71.9 vs 76.9 ms at 3) -- tools/exp_p1x2*.sh
#ifndef BSIDMAP_SCALAR_MN_MAX
#define BSIDMAP_SCALAR_MN_MAX 20
#endif
#ifndef BSIDMAP_L1C_MINB_LOW
#define BSIDMAP_L1C_MINB_LOW 3
#endif
#ifndef BSIDMAP_L1C_MINB
#define BSIDMAP_L1C_MINB \
  (Core::kMinBlocks > 2 ? 4 : (Core::Mn <= BSIDMAP_SCALAR_MN_MAX ? BSIDMAP_L1C_MINB_LOW : Core::kMinBlocks))
#endif
// row pairs (ILP) in pass 1 only where the register budget allows 3 CTAs/SM
#ifndef BSIDMAP_L1_GROUP
#define BSIDMAP_L1_GROUP (Core::kMinBlocks > 2 ? 2 : 1)
#endif
template <class Core, bool kStoreGamma>
__global__ void __launch_bounds__(kLatticeThreads, BSIDMAP_L1_MINB) k_gamma_sum_x2(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  extern __shared__ uint32_t s_C[];
  const int i = blockIdx.y + p.i_base;
  for (int t = threadIdx.x; t < p.q; t += blockDim.x) s_C[t] = p.C[(size_t)i * p.q + t];
  __syncthreads();

  const long ga = (long)blockIdx.x * (2 * blockDim.x) + threadIdx.x;
  const LaneGeom A = lane_geom_at(p, i, ga), B = lane_geom_at(p, i, ga + blockDim.x);
  f32x2 acc[MN];
#pragma unroll
  for (int e = 0; e < MN; e++) acc[e] = 0ull;

  if (__any_sync(0xffffffffu, A.active || B.active)) {
    typename Core::Lane lane;
    Core::init(lane, A.active ? load_window(p, A.f, A.s, A.rho) : 0ull,
               B.active ? load_window(p, B.f, B.s, B.rho) : 0ull, p);
    const float* pa = p.priors ? p.priors + ((size_t)A.f * p.N + i) * p.q : nullptr;
    const float* pb = p.priors ? p.priors + ((size_t)B.f * p.N + i) * p.q : nullptr;
    const float usc = 1.f / p.q;
    for (int D = 0; D < p.q; D++) {
      const f32x2 P = pa ? pk(__ldg(pa + D), __ldg(pb + D)) : pk(1.f, 1.f);
      f32x2 fo[MN];
      Core::template run<BSIDMAP_L1_GROUP>(lane, s_C[D], p, fo);
#pragma unroll
      for (int e = 0; e < MN; e++) acc[e] = ffma2(P, fo[e], acc[e]);
      if constexpr (kStoreGamma) {
        const float sa = pa ? lo_of(P) : usc, sb = pa ? hi_of(P) : usc;
        if (A.in) {
          float* g = p.gamma + ((((size_t)A.f * p.N + i) * p.q + D) * MN) * p.Mt + A.mi;
#pragma unroll
          for (int e = 0; e < MN; e++) __stcs(g + (size_t)e * p.Mt, out_valid(p, A, e) ? sa * lo_of(fo[e]) : 0.f);
        }
        if (B.in) {
          float* g = p.gamma + ((((size_t)B.f * p.N + i) * p.q + D) * MN) * p.Mt + B.mi;
#pragma unroll
          for (int e = 0; e < MN; e++) __stcs(g + (size_t)e * p.Mt, out_valid(p, B, e) ? sb * hi_of(fo[e]) : 0.f);
        }
      }
    }
  } else if constexpr (kStoreGamma) {
    for (int w = 0; w < 2; w++) {
      const LaneGeom& G = w ? B : A;
      if (!G.in) continue;
      float* g = p.gamma + (((size_t)G.f * p.N + i) * p.q) * MN * p.Mt + G.mi;
      for (int D = 0; D < p.q; D++)
#pragma unroll
        for (int e = 0; e < MN; e++) __stcs(g + ((size_t)D * MN + e) * p.Mt, 0.f);
    }
  }
  const float sc = p.priors ? 1.f : 1.f / p.q;
  if (A.in) {
    float* out = p.Gsum + ((size_t)A.f * p.N + i) * MN * p.Mtp + A.mi;
#pragma unroll
    for (int e = 0; e < MN; e++) out[(size_t)e * p.Mtp] = out_valid(p, A, e) ? sc * lo_of(acc[e]) : 0.f;
  }
  if (B.in) {
    float* out = p.Gsum + ((size_t)B.f * p.N + i) * MN * p.Mtp + B.mi;
#pragma unroll
    for (int e = 0; e < MN; e++) out[(size_t)e * p.Mtp] = out_valid(p, B, e) ? sc * hi_of(acc[e]) : 0.f;
  }
}

// ---------------------------------------------------------------------------------------
// Pass 1 with the last K lattice rows hoisted out of the symbol loop.  The rows are linear in
// the row they read and rows n-K+1..n depend only on the codeword's last K bits, so
//   Gamma_i(m', .) = sum_cls Last_cls( sum_{D : C_i(D) ends in cls} P(D) G_{n-K}(m', ., D) ):
// the symbols are visited class by class (C_i grouped by its last K bits once at create: Cs/Ds/Cst)
// and the last K rows run once per class instead of once per symbol.  Exact algebra; the
// node count of the algorithm is unchanged (the roofline still counts 5 flops per node).
// Symbol indices per CTA of the pass-1 kernels: the windows' frame geometry is loaded once and the
// received words of step i + 1 are prefetched while step i computes.
#ifndef BSIDMAP_L1_STEPS
#define BSIDMAP_L1_STEPS 8
#endif
constexpr int kL1Steps = BSIDMAP_L1_STEPS;

__device__ __forceinline__ LaneGeom geom_step(const DecodeParams& p, const WinBase& b, int i) {
  LaneGeom G;
  G.in = b.in;
  G.f = b.f;
  G.mi = b.mi;
  G.mp = b.mp;
  G.s = p.n * i + b.mp;  // window start n i + m' (eqn:gamma)
  G.rho = b.rho;
  G.active = b.ok && G.s >= 0 && G.s <= G.rho;
  G.vmask = valid_mask(p, G);
  return G;
}

template <class Core, int K, bool kPri = true>
__global__ void __launch_bounds__(kLatticeThreads, BSIDMAP_L1C_MINB) k_gamma_sum_x2_cls(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  constexpr int NC = 1 << K;
  extern __shared__ __align__(128) unsigned char smem[];
  f32x2* s_res = reinterpret_cast<f32x2*>(smem);  // [MN][128] per-lane result (private column, no barrier)
  const long ga = (long)blockIdx.x * (2 * blockDim.x) + threadIdx.x;
  const WinBase ba = win_base(p, ga), bb = win_base(p, ga + blockDim.x);
  const int i0 = p.i_base + blockIdx.y * p.i_steps, i1 = min(i0 + p.i_steps, p.i_end);
  Win3 na = win_words(ba, p.n * i0 + ba.mp), nb = win_words(bb, p.n * i0 + bb.mp);
#pragma unroll 1
  for (int i = i0; i < i1; i++) {
    const LaneGeom A = geom_step(p, ba, i), B = geom_step(p, bb, i);
    const Win3 wa = na, wb = nb;
    if (i + 1 < i1) {  // prefetch the next step's received words
      na = win_words(ba, A.s + p.n);
      nb = win_words(bb, B.s + p.n);
    }
    const uint32_t* Ci = p.Cs[K - 2] + (size_t)i * p.q;  // C_i grouped by the class of its last K bits
    const uint16_t* Di = p.Ds[K - 2] + (size_t)i * p.q;
    f32x2 acc[MN];
#pragma unroll
    for (int e = 0; e < MN; e++) acc[e] = 0ull;
    if (__any_sync(0xffffffffu, A.active || B.active)) {
      typename Core::Lane lane;
      Core::init(lane, A.active ? win_bits(wa, A.s) : 0ull, B.active ? win_bits(wb, B.s) : 0ull, p);
      const float* pa = p.priors ? p.priors + ((size_t)A.f * p.N + i) * p.q : nullptr;
      const float* pb = p.priors ? p.priors + ((size_t)B.f * p.N + i) * p.q : nullptr;
      f32x2* res = s_res + threadIdx.x;  // res[e * 128]: the sum over the finished classes
      bool first = true;
      const int sh = p.n - K;
      XPrefetch xs(Ci, 0, p.q);
      uint32_t cur = (Ci[0] >> sh) & (NC - 1);
      // one pass over C_i in class order; the class boundary is seen in the (warp-uniform) codeword
      for (int k = 0; k < p.q; k++) {
        const uint32_t x = xs.take(k);
        const uint32_t c = (x >> sh) & (NC - 1);
        if (c != cur) {  // close class `cur`: its last K rows once, added to the finished classes
          Core::template apply_last_rows<K>(lane, cur, p, acc);
#pragma unroll
          for (int e = 0; e < MN; e++) {
            if (!first) acc[e] = fadd2(acc[e], res[e * kLatticeThreads]);
            res[e * kLatticeThreads] = acc[e];
            acc[e] = 0ull;
          }
          first = false;
          cur = c;
        }
        f32x2 fo[MN];
        f32x2 P = 0ull;
        if constexpr (kPri) {  // P(D_i = D) of the two windows' frames
          const int D = Di[k];
          P = pk(__ldg(pa + D), __ldg(pb + D));
        }
        auto add = [&](const f32x2 (&g)[MN]) {
#pragma unroll
          for (int e = 0; e < MN; e++) acc[e] = kPri ? ffma2(P, g[e], acc[e]) : fadd2(g[e], acc[e]);
        };
        // the class-sum update inside the last row group's basic block (rows_then); uniform priors:
        // the common factor 1/q is applied at the store
        Core::template run_prefix_then<K, BSIDMAP_L1_GROUP>(lane, x, p, fo, add);
      }
      Core::template apply_last_rows<K>(lane, cur, p, acc);
      if (!first) {
#pragma unroll
        for (int e = 0; e < MN; e++) acc[e] = fadd2(acc[e], res[e * kLatticeThreads]);
      }
    }
    const float sc = p.priors ? 1.f : 1.f / p.q;
    if (A.in) {
      float* out = p.Gsum + ((size_t)A.f * p.N + i) * MN * p.Mtp + A.mi;
#pragma unroll
      for (int e = 0; e < MN; e++) out[(size_t)e * p.Mtp] = out_valid(p, A, e) ? sc * lo_of(acc[e]) : 0.f;
    }
    if (B.in) {
      float* out = p.Gsum + ((size_t)B.f * p.N + i) * MN * p.Mtp + B.mi;
#pragma unroll
      for (int e = 0; e < MN; e++) out[(size_t)e * p.Mtp] = out_valid(p, B, e) ? sc * hi_of(acc[e]) : 0.f;
    }
  }
}

// Scalar-core version (one window per lane, flat geometry) for the register-heavy shapes.
template <class Core, int K, bool kPri = true>
__global__ void __launch_bounds__(kLatticeThreads, kLatticeMinBlocks) k_gamma_sum_cls(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  constexpr int NC = 1 << K;
  extern __shared__ __align__(128) unsigned char smem[];
  float* s_res = reinterpret_cast<float*>(smem);  // [MN][128] per-lane result (private column, no barrier)
  const WinBase wb = win_base(p, (long)blockIdx.x * blockDim.x + threadIdx.x);
  const int i0 = p.i_base + blockIdx.y * p.i_steps, i1 = min(i0 + p.i_steps, p.i_end);
  Win3 nw = win_words(wb, p.n * i0 + wb.mp);
#pragma unroll 1
  for (int i = i0; i < i1; i++) {
    const LaneGeom G = geom_step(p, wb, i);
    const Win3 ww = nw;
    if (i + 1 < i1) nw = win_words(wb, G.s + p.n);  // prefetch the next step's received words
    const uint32_t* Ci = p.Cs[K - 2] + (size_t)i * p.q;
    const uint16_t* Di = p.Ds[K - 2] + (size_t)i * p.q;
    const int* cst = p.Cst[K - 2] + (size_t)i * (NC + 1);
    float acc[MN];
#pragma unroll
    for (int e = 0; e < MN; e++) acc[e] = 0.f;
    if (__any_sync(0xffffffffu, G.active)) {
      typename Core::Lane lane;
      Core::init(lane, G.active ? win_bits(ww, G.s) : 0ull, p);
      const float* pri = p.priors ? p.priors + ((size_t)G.f * p.N + i) * p.q : nullptr;
      float* res = s_res + threadIdx.x;  // the sum over the finished classes
      bool first = true;
      int k = 0;
      XPrefetch xs(Ci, 0, p.q);
      // class by class (measured faster than the single loop of k_gamma_sum_x2_cls for this core)
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
          if (!first) acc[e] += res[e * kLatticeThreads];
          res[e * kLatticeThreads] = acc[e];
        }
        first = false;
      }
    }
    if (G.in) {
      const float sc = p.priors ? 1.f : 1.f / p.q;
      float* out = p.Gsum + ((size_t)G.f * p.N + i) * MN * p.Mtp + G.mi;
#pragma unroll
      for (int e = 0; e < MN; e++) out[(size_t)e * p.Mtp] = out_valid(p, G, e) ? sc * acc[e] : 0.f;
    }
  }
}

// beta_{i+1}(m'+k) of one window, scaled by 2^-E (E = exponent of its corridor max),
// as FP32 in [0, 2); returns w = alpha_i(m') 2^E (FP64) so that w * bt = alpha * beta exactly.
template <int MN>
__device__ __forceinline__ double app_weights_p2(const DecodeParams& p, const LaneGeom& G, int i, float (&bt)[MN]) {
  double bv[MN];
  double bm = 0.0;
  const double* brow = p.beta + ((size_t)G.f * (p.N + 1) + (i + 1)) * p.Mt;
  const int m0 = G.mi + p.mn_lo;
#pragma unroll
  for (int e = 0; e < MN; e++) {
    const double v = __ldg(brow + min(max(m0 + e, 0), p.Mt - 1));  // clamped: all loads in flight together
    bv[e] = ((G.vmask >> e) & 1u) ? v : 0.0;
    bm = fmax(bm, bv[e]);
  }
  const int E = bm > 0.0 ? exp2_of(bm) : 0;
  const double sc = pow2d(-E);
#pragma unroll
  for (int e = 0; e < MN; e++) bt[e] = (float)(bv[e] * sc);
  return (G.active && bm > 0.0) ? p.alpha[((size_t)G.f * (p.N + 1) + i) * p.Mt + G.mi] * pow2d(E) : 0.0;
}

// The same for the two windows m'_a = m', m'_b = m' + 1 of a lane (B.mi = A.mi + 1): their
// corridors share M_n - 1 states, so M_n + 1 loads serve both; the corridor maximum's exponent
// comes from the high words (for doubles >= 0 the integer order of the high word is the order
// of the value's exponent), one integer max per state instead of an FP64 compare-and-select.
template <int MN>
__device__ __forceinline__ void app_weights_pair(const DecodeParams& p, const LaneGeom& A, const LaneGeom& B, int i,
                                                 float (&ba)[MN], float (&bb)[MN], double& da, double& db) {
  double bv[MN + 1];
  const double* brow = p.beta + ((size_t)A.f * (p.N + 1) + (i + 1)) * p.Mt;
  const int m0 = A.mi + p.mn_lo;
#pragma unroll
  for (int u = 0; u < MN + 1; u++) bv[u] = __ldg(brow + min(max(m0 + u, 0), p.Mt - 1));
  int ha = 0, hb = 0;
#pragma unroll
  for (int e = 0; e < MN; e++) {
    if ((A.vmask >> e) & 1u) ha = max(ha, __double2hiint(bv[e]));
    if ((B.vmask >> e) & 1u) hb = max(hb, __double2hiint(bv[e + 1]));
  }
  const int Ea = ha > 0 ? (ha >> 20) - 1023 : 0, Eb = hb > 0 ? (hb >> 20) - 1023 : 0;
  const double sa = pow2d(-Ea), sb = pow2d(-Eb);
#pragma unroll
  for (int e = 0; e < MN; e++) {
    ba[e] = ((A.vmask >> e) & 1u) ? (float)(bv[e] * sa) : 0.f;
    bb[e] = ((B.vmask >> e) & 1u) ? (float)(bv[e + 1] * sb) : 0.f;
  }
  const double* arow = p.alpha + ((size_t)A.f * (p.N + 1) + i) * p.Mt;
  da = (A.active && ha > 0) ? arow[A.mi] * pow2d(Ea) : 0.0;
  db = (B.active && hb > 0) ? arow[B.mi] * pow2d(Eb) : 0.0;
}

// APP pass: 5 CTAs/SM (102 registers; the beta corridor lives in smem) with row pairs measured
// fastest on B200 for C2 (tools/exp_app.sh: 17.06 ms vs 17.3-18.0 ms for 3-4 CTAs/SM)
#ifndef BSIDMAP_APP_MINB
#define BSIDMAP_APP_MINB (Core::kMinBlocks > 2 ? 5 : 2)
#endif
#ifndef BSIDMAP_APP_GROUP
#define BSIDMAP_APP_GROUP (Core::kMinBlocks > 2 ? 2 : 1)
#endif
// per-warp staging of the per-lane contributions c(lane, D): [q][33] floats (odd stride), reduced
// over the lanes once after the D loop instead of one shuffle chain per D
__host__ __device__ __forceinline__ size_t app_stage_floats(int q) { return (size_t)q * 33; }
__host__ __device__ __forceinline__ size_t app_x2_smem(int q, int Mn, int ks = 1) {
  return (size_t)kX2Warps * (2 << (ks - 1)) * Mn * 32 * 8 + (size_t)kX2Warps * (app_stage_floats(q) * 4 + (size_t)q * 8);
}
// Symbols are visited in lexicographic codeword order (DecodeParams::Cp, prepared at create) so
// that lattice rows 1..KP (run_head) are computed once per distinct prefix; KP = 0: natural order.
// The prefix length that saves the most nodes for random codebooks: ~log2(q) - 1.
__host__ __device__ __forceinline__ int app_prefix_bits(int q, int n) {
  int kp = q <= 8 ? 2 : q <= 16 ? 3 : 4;
  return kp <= n - 2 ? kp : 0;
}
// smem: s_w[kX2Warps][2][M_n][32] (f32x2: the scaled beta corridor of each lane's two windows with
//       the last lattice row folded in, one table per value of x_n; smem, not registers) |
//       s_S[kX2Warps][q] (double) | staging [kX2Warps][q][33] (float)
// prefix sharing keeps the head row live across the symbol loop (+2 M_n registers)
#ifndef BSIDMAP_APP_MINB_PRE
#define BSIDMAP_APP_MINB_PRE (Core::kMinBlocks > 2 ? 4 : 2)
#endif
// KS = lattice rows folded into the APP weights: 1 = the last row (two tables, by x_n); 2 = the
// last two rows (four tables, by (x_{n-1}, x_n); row n-1 transposed by SpecCoreX2::row_transpose),
// so each symbol runs rows 1..n-2 only.  Exact re-association (the rows are linear maps).
// the weight dot inside the basic block of the last lattice row (rows_then), so it interleaves
// with the row's insertion chain instead of running as a dependent tail after the branch merge
#ifndef BSIDMAP_APP_MINB_KS2
#define BSIDMAP_APP_MINB_KS2 (Core::kMinBlocks > 2 ? 3 : 2)
#endif
template <class Core, int KP, int KS = 1>
__global__ void __launch_bounds__(kLatticeThreads, KS == 2 ? BSIDMAP_APP_MINB_KS2
                                                           : (KP > 0 ? BSIDMAP_APP_MINB_PRE : BSIDMAP_APP_MINB))
    k_app_x2(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  constexpr int NT = 2 << (KS - 1);  // weight tables per lane
  constexpr int RL = Core::NNr - KS;  // last lattice row run per symbol
  extern __shared__ __align__(128) unsigned char smem[];
  f32x2* s_bt = reinterpret_cast<f32x2*>(smem);
  double* s_S = reinterpret_cast<double*>(s_bt + kX2Warps * NT * MN * 32);
  float* s_stage = reinterpret_cast<float*>(s_S + kX2Warps * p.q);
  const int i = blockIdx.y + p.i_base;
  // KP > 0: symbols in lexicographic codeword order (prefix groups contiguous); every smem array
  // below is per warp, so the kernel has no block barrier
  const uint32_t* Ci = (KP > 0 ? p.Cp : p.C) + (size_t)i * p.q;
  const uint16_t* Di = p.Dp + (size_t)i * p.q;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = tiles_per_frame(p.Mt);
  const long tile = (long)blockIdx.x * kX2Warps + warp;
  const int f = (int)(tile / T);
  if (f >= p.F) return;  // warp-uniform; no block barrier follows
  const int mia = (int)(tile % T) * kTileSlots + 2 * lane;
  const LaneGeom A = geom_fm(p, i, f, mia, mia < p.Mt);
  const LaneGeom B = geom_fm(p, i, f, mia + 1, mia + 1 < p.Mt);
  const bool frame_ok = p.status[f] == kFrameOk;

  // KS = 1: w1[e] at wt[e*32], w0[e] at wt[(MN+e)*32]; KS = 2: table c = 2 [x_n = 0] + [x_{n-1} = 0]
  f32x2* wt = s_bt + (size_t)warp * NT * MN * 32 + lane;
  float wa, wb;
  int Emax;
  f32x2 bt[MN];
  {
    float ba[MN], bb[MN];
    double da, db;
    app_weights_pair<MN>(p, A, B, i, ba, bb, da, db);
#pragma unroll
    for (int e = 0; e < MN; e++) bt[e] = pk(ba[e], bb[e]);
    // common power-of-two scale of the tile's weights (max exponent over the warp)
    const double dm = fmax(da, db);
    Emax = __reduce_max_sync(0xffffffffu, dm > 0.0 ? exp2_of(dm) + 2048 : 0) - 2048;
    const double sc = pow2d(-Emax);
    wa = (float)(da * sc);
    wb = (float)(db * sc);
  }
  const bool live = __any_sync(0xffffffffu, wa > 0.f || wb > 0.f);
  double* S = s_S + warp * p.q;
  float* stg = s_stage + (size_t)warp * app_stage_floats(p.q);
  if (live) {
    typename Core::Lane lane_t;
    Core::init(lane_t, A.active ? load_window(p, A.f, A.s, A.rho) : 0ull,
               B.active ? load_window(p, B.f, B.s, B.rho) : 0ull, p);
    if constexpr (KS == 1) {
      Core::last_row_weights(lane_t, [&](int e) { return bt[e]; }, [&](int e) -> f32x2& { return wt[e * 32]; },
                             [&](int e) -> f32x2& { return wt[(MN + e) * 32]; });
    } else {
      f32x2 w1[MN], w0[MN], wi[MN];
      Core::last_row_weights(lane_t, [&](int e) { return bt[e]; }, [&](int e) -> f32x2& { return w1[e]; },
                             [&](int e) -> f32x2& { return w0[e]; });
      const f32x2 a2 = pk(p.lc.a, p.lc.a);
      Core::template row_transpose<Core::NNr - 1>(w1, wi, lane_t.q1, a2);  // (x_{n-1}, x_n) = (1, 1)
#pragma unroll
      for (int e = 0; e < MN; e++) wt[e * 32] = wi[e];
      Core::template row_transpose<Core::NNr - 1>(w1, wi, lane_t.q0, a2);  // (0, 1)
#pragma unroll
      for (int e = 0; e < MN; e++) wt[(MN + e) * 32] = wi[e];
      Core::template row_transpose<Core::NNr - 1>(w0, wi, lane_t.q1, a2);  // (1, 0)
#pragma unroll
      for (int e = 0; e < MN; e++) wt[(2 * MN + e) * 32] = wi[e];
      Core::template row_transpose<Core::NNr - 1>(w0, wi, lane_t.q0, a2);  // (0, 0)
#pragma unroll
      for (int e = 0; e < MN; e++) wt[(3 * MN + e) * 32] = wi[e];
    }
    const float* pri = p.priors ? p.priors + ((size_t)f * p.N + i) * p.q : nullptr;
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
      f32x2 t0 = 0ull, t1 = 0ull;
      auto dot = [&](const f32x2 (&g)[MN]) {
#pragma unroll
        for (int e = 0; e < MN; e += 2) {
          t0 = ffma2(g[e], W[e * 32], t0);
          if (e + 1 < MN) t1 = ffma2(g[e + 1], W[(e + 1) * 32], t1);
        }
      };
      if constexpr (KP > 0) {
        if (k == 0 || ((x ^ xprev) & ((1u << KP) - 1u)) != 0u)
          Core::template run_head<KP, BSIDMAP_APP_GROUP>(lane_t, x, p, fh);
        xprev = x;
#pragma unroll
        for (int e = 0; e < MN; e++) fo[e] = fh[e];
        Core::template run_tail_to_then<KP, RL, BSIDMAP_APP_GROUP>(lane_t, x, p, fo, dot);
      } else {
        Core::template run_to_then<RL, BSIDMAP_APP_GROUP>(lane_t, x, p, fo, dot);
      }
      const int D = KP > 0 ? (int)Di[k] : k;
      stg[D * 33 + lane] = fmaf(wa, lo_of(t0) + lo_of(t1), wb * (hi_of(t0) + hi_of(t1)));
    }
    __syncwarp();
    for (int D = lane; D < p.q; D += 32) {  // S(D) = P(D) sum over the warp's windows (FP64)
      double c = 0.0;
#pragma unroll 8
      for (int l = 0; l < 32; l++) c += (double)stg[D * 33 + l];
      S[D] = pri ? c * (double)__ldg(pri + D) : c;
    }
  }
  __syncwarp();
  if (T == 1) {
    // the warp holds the whole sum over m': L_i(D) = S(D) / sum_D S(D)
    double tot = 0.0;
    if (live)
      for (int D = lane; D < p.q; D += 32) tot += S[D];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    const bool ok = frame_ok && live && tot > 0.0;
    const double inv = ok ? 1.0 / tot : 0.0;
    float* Lrow = p.L + ((size_t)f * p.N + i) * p.q;
    for (int D = lane; D < p.q; D += 32) Lrow[D] = ok ? (float)(S[D] * inv) : 0.f;
    if (frame_ok && !ok && lane == 0) p.status[f] = kFrameUnderflow;
  } else if (live) {
    const double sc = pow2d(Emax);
    double* acc = p.Lacc + ((size_t)f * p.N + i) * p.q;
    for (int D = lane; D < p.q; D += 32) {
      const double v = S[D];
      if (v > 0.0) atomicAdd(acc + D, v * sc);
    }
  }
}

// Scalar-core APP on frame-aligned 32-state warp tiles (one window per lane): used where the
// pair core is register-bound (C3, C5) -- also wastes fewer slots (C3: 9 x 32 vs 5 x 64 for 267).
__host__ __device__ __forceinline__ int tiles_per_frame_w(int Mt, int W) { return (Mt + 32 * W - 1) / (32 * W); }
__host__ __device__ __forceinline__ size_t app_x1_smem(int q, int Mn = 0, int ks = 1) {
  return (size_t)kX2Warps * (app_stage_floats(q) * 4 + (size_t)q * 8) + (ks == 2 ? (size_t)4 * Mn * kLatticeThreads * 4 : 0);
}

#ifndef BSIDMAP_APP1_MINB_PRE
#define BSIDMAP_APP1_MINB_PRE 3
#endif
// KS = 2: the last two rows folded into four per-lane weight tables in shared memory (see k_app_x2)
template <class Core, int KP, int KS = 1>
__global__ void __launch_bounds__(kLatticeThreads, (KP > 0 || KS == 2) ? BSIDMAP_APP1_MINB_PRE : kLatticeMinBlocks)
    k_app_x1(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  constexpr int RL = Core::NNr - KS;  // last lattice row run per symbol
  extern __shared__ __align__(128) unsigned char smem[];
  double* s_S = reinterpret_cast<double*>(smem);
  float* s_stage = reinterpret_cast<float*>(s_S + kX2Warps * p.q);
  float* s_w = s_stage + (size_t)kX2Warps * app_stage_floats(p.q) + threadIdx.x;  // KS = 2: [4][MN][128]
  const int i = blockIdx.y + p.i_base;
  const uint32_t* Ci = (KP > 0 ? p.Cp : p.C) + (size_t)i * p.q;
  const uint16_t* Di = p.Dp + (size_t)i * p.q;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = tiles_per_frame_w(p.Mt, 1);
  const long tile = (long)blockIdx.x * kX2Warps + warp;
  const int f = (int)(tile / T);
  if (f >= p.F) return;  // warp-uniform; no block barrier follows
  const int mi = (int)(tile % T) * 32 + lane;
  const LaneGeom A = geom_fm(p, i, f, mi, mi < p.Mt);
  const bool frame_ok = p.status[f] == kFrameOk;
  float bt[MN];
  float wa;
  int Emax;
  {
    const double da = app_weights_p2<MN>(p, A, i, bt);  // bt: corridor weights (see app_weights_p2)
    Emax = __reduce_max_sync(0xffffffffu, da > 0.0 ? exp2_of(da) + 2048 : 0) - 2048;
    wa = (float)(da * pow2d(-Emax));
  }
  const bool live = __any_sync(0xffffffffu, wa > 0.f);
  double* S = s_S + warp * p.q;
  float* stg = s_stage + (size_t)warp * app_stage_floats(p.q);
  if (live) {
    typename Core::Lane lane_t;
    Core::init(lane_t, A.active ? load_window(p, A.f, A.s, A.rho) : 0ull, p);
    float w1[MN], w0[MN];  // last lattice row folded into the weights (one table per x_n)
    Core::last_row_weights(lane_t, bt, w1, w0);
    if constexpr (KS == 2) {  // table c = 2 [x_n = 0] + [x_{n-1} = 0], entry e at s_w[(c MN + e) 128]
      float wi[MN];
      Core::template row_transpose<Core::NNr - 1>(w1, wi, lane_t.q1, p.lc.a);
#pragma unroll
      for (int e = 0; e < MN; e++) s_w[e * kLatticeThreads] = wi[e];
      Core::template row_transpose<Core::NNr - 1>(w1, wi, lane_t.q0, p.lc.a);
#pragma unroll
      for (int e = 0; e < MN; e++) s_w[(MN + e) * kLatticeThreads] = wi[e];
      Core::template row_transpose<Core::NNr - 1>(w0, wi, lane_t.q1, p.lc.a);
#pragma unroll
      for (int e = 0; e < MN; e++) s_w[(2 * MN + e) * kLatticeThreads] = wi[e];
      Core::template row_transpose<Core::NNr - 1>(w0, wi, lane_t.q0, p.lc.a);
#pragma unroll
      for (int e = 0; e < MN; e++) s_w[(3 * MN + e) * kLatticeThreads] = wi[e];
    }
    const float* pri = p.priors ? p.priors + ((size_t)f * p.N + i) * p.q : nullptr;
    const int nb = p.n - 1;
    float fh[MN];  // rows 1..KP of the current prefix
    XPrefetch xs(Ci, 0, p.q);
    uint32_t xprev = 0u;
    for (int k = 0; k < p.q; k++) {
      const uint32_t x = xs.take(k);
      const int D = KP > 0 ? (int)Di[k] : k;
      float fo[MN];
      float t0 = 0.f, t1 = 0.f;
      // KS = 2: the table dot fused into the last row's basic block (rows_then); KS = 1: after it
      const float* W = s_w + (size_t)((((x >> nb) & 1u) ? 0 : 2) + (((x >> (nb - 1)) & 1u) ? 0 : 1)) * MN * kLatticeThreads;
      auto dot = [&](const float (&g)[MN]) {
        if constexpr (KS == 2) {
#pragma unroll
          for (int e = 0; e < MN; e += 2) {
            t0 = fmaf(g[e], W[e * kLatticeThreads], t0);
            if (e + 1 < MN) t1 = fmaf(g[e + 1], W[(e + 1) * kLatticeThreads], t1);
          }
        }
      };
      if constexpr (KP > 0) {
        if (k == 0 || ((x ^ xprev) & ((1u << KP) - 1u)) != 0u) Core::template run_head<KP>(lane_t, x, p, fh);
        xprev = x;
#pragma unroll
        for (int e = 0; e < MN; e++) fo[e] = fh[e];
        if constexpr (KS == 2) Core::template run_tail_to_then<KP, RL>(lane_t, x, p, fo, dot);
        else Core::template run_tail_to<KP, RL>(lane_t, x, p, fo);
      } else {
        if constexpr (KS == 2) Core::template run_to_then<RL>(lane_t, x, p, fo, dot);
        else Core::template run_to<RL>(lane_t, x, p, fo);
      }
      if constexpr (KS == 2) {
      } else if ((x >> nb) & 1u) {
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
      stg[D * 33 + lane] = wa * (t0 + t1);
    }
    __syncwarp();
    for (int D = lane; D < p.q; D += 32) {  // FP64, as k_app_x2
      double c = 0.0;
#pragma unroll 8
      for (int l = 0; l < 32; l++) c += (double)stg[D * 33 + l];
      S[D] = pri ? c * (double)__ldg(pri + D) : c;
    }
  }
  __syncwarp();
  if (T == 1) {
    double tot = 0.0;
    if (live)
      for (int D = lane; D < p.q; D += 32) tot += S[D];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    const bool ok = frame_ok && live && tot > 0.0;
    const double inv = ok ? 1.0 / tot : 0.0;
    float* Lrow = p.L + ((size_t)f * p.N + i) * p.q;
    for (int D = lane; D < p.q; D += 32) Lrow[D] = ok ? (float)(S[D] * inv) : 0.f;
    if (frame_ok && !ok && lane == 0) p.status[f] = kFrameUnderflow;
  } else if (live) {
    const double sc = pow2d(Emax);
    double* acc = p.Lacc + ((size_t)f * p.N + i) * p.q;
    for (int D = lane; D < p.q; D += 32) {
      const double v = S[D];
      if (v > 0.0) atomicAdd(acc + D, v * sc);
    }
  }
}

template <class Core>
__global__ void __launch_bounds__(kLatticeThreads) k_gamma_dump_x2(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  extern __shared__ uint32_t s_C[];
  const int i = p.dbg_i;
  for (int t = threadIdx.x; t < p.q; t += blockDim.x) s_C[t] = p.C[(size_t)i * p.q + t];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = tiles_per_frame(p.Mt);
  const long tile = (long)blockIdx.x * kX2Warps + warp;
  const int f = (int)(tile / T);
  const int mia = (int)(tile % T) * kTileSlots + 2 * lane;
  const LaneGeom A = geom_fm(p, i, f, mia, f < p.F && mia < p.Mt);
  const LaneGeom B = geom_fm(p, i, f, mia + 1, f < p.F && mia + 1 < p.Mt);
  typename Core::Lane lane_t;
  Core::init(lane_t, A.active ? load_window(p, A.f, A.s, A.rho) : 0ull,
             B.active ? load_window(p, B.f, B.s, B.rho) : 0ull, p);
  const double unscale = p.lc.out_scale;
  for (int D = 0; D < p.q; D++) {
    f32x2 fo[MN];
    Core::run(lane_t, s_C[D], p, fo);
    for (int w = 0; w < 2; w++) {
      const LaneGeom& G = w ? B : A;
      if (!G.in) continue;
      const double P = p.priors ? (double)p.priors[((size_t)G.f * p.N + i) * p.q + D] : 1.0 / p.q;
      double* out = p.dbg_gamma + ((size_t)G.f * p.Mt + G.mi) * MN * p.q;
#pragma unroll
      for (int e = 0; e < MN; e++)
        out[(size_t)e * p.q + D] = out_valid(p, G, e) ? P * (double)(w ? hi_of(fo[e]) : lo_of(fo[e])) * unscale : 0.0;
    }
  }
}

template <class Core>
CoreKernels make_core_kernels_x2(long nodes);  // defined in k_local_x2.cuh (needs the local kernels)
}  // namespace bsidmap
#include "k_app_live.cuh"
namespace bsidmap {

template <class Core>
CoreKernels make_core_kernels_x2_base(long nodes) {
  CoreKernels k{};
  k.gamma_sum = k_gamma_sum_x2_cls<Core, 2, false>;
  k.gamma_sum_k3 = k_gamma_sum_x2_cls<Core, 3, false>;
  k.gamma_sum_pri = k_gamma_sum_x2_cls<Core, 2, true>;
  k.gamma_sum_k3_pri = k_gamma_sum_x2_cls<Core, 3, true>;
  k.gamma_store = k_gamma_sum_x2<Core, true>;
  k.app = k_app_x2<Core, 0>;
  k.app_pre[0] = k_app_x2<Core, 2>;
  k.app_pre[1] = k_app_x2<Core, 3>;
  k.app_pre[2] = k_app_x2<Core, 4>;
  k.app_ks2 = k_app_x2<Core, 0, 2>;
  k.app_ks_auto = Core::kMinBlocks <= 2 ? 2 : 1;
  k.app_pre_ks2[0] = k_app_x2<Core, 2, 2>;
  k.app_pre_ks2[1] = k_app_x2<Core, 3, 2>;
  k.app_pre_ks2[2] = k_app_x2<Core, 4, 2>;
  k.app_live[0][0] = k_app_live_x2<Core, 0, 1>;
  k.app_live[0][1] = k_app_live_x2<Core, 2, 1>;
  k.app_live[0][2] = k_app_live_x2<Core, 3, 1>;
  k.app_live[0][3] = k_app_live_x2<Core, 4, 1>;
  k.app_live[1][0] = k_app_live_x2<Core, 0, 2>;
  k.app_live[1][1] = k_app_live_x2<Core, 2, 2>;
  k.app_live[1][2] = k_app_live_x2<Core, 3, 2>;
  k.app_live[1][3] = k_app_live_x2<Core, 4, 2>;
  k.app_live_W = 2;
  k.app_stored = k_app_stored<Core::Mn>;
  k.gamma_dump = k_gamma_dump_x2<Core>;
  k.nodes = nodes;
  k.W = 2;
  k.l1_W = 2;
  k.l1_steps = true;
  k.app_W = 2;
  k.ab_warp[0] = k_alpha_beta_warp<1, Core::Mn>;
  k.ab_warp[1] = k_alpha_beta_warp<2, Core::Mn>;
  k.ab_warp[2] = k_alpha_beta_warp<4, Core::Mn>;
  return k;
}

}  // namespace bsidmap
