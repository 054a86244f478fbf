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
// row pairs (ILP) in pass 1 where the register budget allows 3 CTAs/SM; the register-heavy shapes
// measured mixed (tools/exp_p1g.sh, r02m: C3 pass 1 59.7 -> 58.4 ms, C5 equal, C4 69.1 -> 72.3,
// J1 143 -> 149), so they keep single rows
#ifndef BSIDMAP_L1_GROUP
#define BSIDMAP_L1_GROUP (Core::kMinBlocks > 2 ? 2 : 1)
#endif
template <class Core, bool kStoreGamma>
__global__ void __launch_bounds__(kLatticeThreads, BSIDMAP_L1_MINB) k_gamma_sum_x2(const DecodeParams p) {
  using f32x2 = typename Core::P2;
  constexpr int MN = Core::Mn;
  extern __shared__ uint32_t s_C[];
  const int i = blockIdx.y + p.i_base;
  for (int t = threadIdx.x; t < p.q; t += blockDim.x) s_C[t] = p.C[(size_t)i * p.q + t];
  __syncthreads();

  const long ga = (long)blockIdx.x * (2 * blockDim.x) + threadIdx.x;
  const LaneGeom A = lane_geom_at(p, i, ga), B = lane_geom_at(p, i, ga + blockDim.x);
  f32x2 acc[MN];
#pragma unroll
  for (int e = 0; e < MN; e++) acc[e] = Core::f2z();

  if (__any_sync(0xffffffffu, A.active || B.active)) {
    typename Core::Lane lane;
    Core::init(lane, A.active ? load_window(p, A.f, A.s, A.rho) : 0ull,
               B.active ? load_window(p, B.f, B.s, B.rho) : 0ull, p);
    const float* pa = p.priors ? p.priors + ((size_t)A.f * p.N + i) * p.q : nullptr;
    const float* pb = p.priors ? p.priors + ((size_t)B.f * p.N + i) * p.q : nullptr;
    const float usc = 1.f / p.q;
    for (int D = 0; D < p.q; D++) {
      const f32x2 P = pa ? Core::pk(__ldg(pa + D), __ldg(pb + D)) : Core::pk(1.f, 1.f);
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
    float* out = gsum_block(p, A.f, i) + A.mi;
#pragma unroll
    for (int e = 0; e < MN; e++) out[(size_t)e * p.Mtp] = out_valid(p, A, e) ? sc * lo_of(acc[e]) : 0.f;
  }
  if (B.in) {
    float* out = gsum_block(p, B.f, i) + B.mi;
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
// Recomputed Gamma (slab schedule, backward sweep, p.askip): a window with alpha_i(m') = 0 contributes
// nothing weighted by a non-zero alpha (reading R19); a warp none of whose windows has alpha != 0
// skips the step and leaves its Gamma rows 0 (windows with alpha = 0 in a warp that runs are computed
// as usual: either value is exact for L).
__device__ __forceinline__ bool alpha_live(const DecodeParams& p, bool askip, const WinBase& b, const LaneGeom& G, int i) {
  return G.active && (!askip || p.alpha[((size_t)b.f * (p.N + 1) + i) * p.Mt + b.mi] != 0.0);
}

// Head tables of pass 1: lattice rows 1..KH depend only on the codeword's first KH bits, so at each
// symbol index the lane computes them once for the 2^KH prefixes (both windows) and keeps row KH of
// each in shared memory (its private column, no barrier); every symbol then starts from its prefix's
// row instead of computing rows 1..KH (and initialising row 0): C2 saves rows 1-2, 17 of its 89
// pass-1 nodes per symbol.  Same operations per node: bit-identical.  KH is the largest of 2, 1, 0
// whose tables (structurally-zero nodes left out) fit beside s_res at the kernel's CTAs per SM.
__host__ __device__ constexpr int l1_head_e0(int R, int LO) { return (R + LO) < 0 ? -(R + LO) : 0; }
__host__ __device__ constexpr size_t l1_head_bytes(int KH, int LO, int MN) {
  return KH == 0 ? 0 : (size_t)(1 << KH) * (size_t)(MN - l1_head_e0(KH, LO)) * kLatticeThreads * 8;
}
__host__ __device__ constexpr int l1_head_rows(int NN, int LO, int MN, int K, int minb) {
  // s_res [MN][128] f32x2 beside the tables; 227 KB per SM shared by minb CTAs, 2 KB margin each
  return (2 <= NN - K && l1_head_bytes(2, LO, MN) + (size_t)MN * kLatticeThreads * 8 + 2048 <= 227u * 1024 / minb) ? 2
       : (1 <= NN - K && l1_head_bytes(1, LO, MN) + (size_t)MN * kLatticeThreads * 8 + 2048 <= 227u * 1024 / minb) ? 1
                                                                                                                   : 0;
}

template <class Core, int K, bool kPri = true>
__global__ void __launch_bounds__(kLatticeThreads, BSIDMAP_L1C_MINB) k_gamma_sum_x2_cls(const DecodeParams p) {
  using f32x2 = typename Core::P2;
  constexpr int MN = Core::Mn;
  constexpr int NC = 1 << K;
  constexpr int KH = l1_head_rows(Core::NNr, Core::Lo, MN, K, BSIDMAP_L1C_MINB);
  constexpr int E0 = l1_head_e0(KH, Core::Lo);
  extern __shared__ __align__(128) unsigned char smem[];
  f32x2* s_res = reinterpret_cast<f32x2*>(smem);  // [MN][128] per-lane result (private column, no barrier)
  f32x2* s_head = s_res + MN * kLatticeThreads + threadIdx.x;  // [2^KH][MN - E0][128]: this lane's column
  // windows g and g + 128 per lane; with the alpha-support skip (slab backward sweep) the packed
  // windows with alpha != 0 of this CTA's symbol indices first, adjacent slots 2t, 2t + 1
  // (win_base_packed): the CTAs past them only write zero rows.  Packing only where it skips more
  // than 1/8 of the windows (C2-C4 have alpha > 0 on 96-98 % of them: the plain geometry, no test).
  const int i0 = p.i_base + blockIdx.y * p.i_steps, i1 = min(i0 + p.i_steps, p.i_end);
  const long g0 = (long)blockIdx.x * (2 * blockDim.x);
  const bool askip = p.askip && 8L * p.spack[(size_t)blockIdx.y * (p.F + 1) + p.F].x < 7L * p.F * p.Mt;
  const long ga = askip ? g0 + 2 * threadIdx.x : g0 + threadIdx.x;
  const long gb = askip ? ga + 1 : ga + blockDim.x;
  const WinBase ba = askip ? win_base_packed(p, ga, blockIdx.y) : win_base(p, ga);
  const WinBase bb = askip ? win_base_packed(p, gb, blockIdx.y) : win_base(p, gb);
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
    for (int e = 0; e < MN; e++) acc[e] = Core::f2z();
    if (__any_sync(0xffffffffu, alpha_live(p, askip, ba, A, i) || alpha_live(p, askip, bb, B, i))) {
      typename Core::Lane lane;
      Core::init(lane, A.active ? win_bits(wa, A.s) : 0ull, B.active ? win_bits(wb, B.s) : 0ull, p);
      if constexpr (KH > 0) {  // rows 1..KH of every prefix, once per symbol index
#pragma unroll 1
        for (int pf = 0; pf < (1 << KH); pf++) {
          f32x2 h[MN];
          Core::template run_head<KH, 1>(lane, (uint32_t)pf, p, h);
#pragma unroll
          for (int e = E0; e < MN; e++) s_head[(pf * (MN - E0) + (e - E0)) * kLatticeThreads] = h[e];
        }
      }
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
            acc[e] = Core::f2z();
          }
          first = false;
          cur = c;
        }
        f32x2 fo[MN];
        f32x2 P = Core::f2z();
        if constexpr (kPri) {  // P(D_i = D) of the two windows' frames
          const int D = Di[k];
          P = Core::pk(__ldg(pa + D), __ldg(pb + D));
        }
        auto add = [&](const f32x2 (&g)[MN]) {
#pragma unroll
          for (int e = 0; e < MN; e++) acc[e] = kPri ? ffma2(P, g[e], acc[e]) : fadd2(g[e], acc[e]);
        };
        // the class-sum update inside the last row group's basic block (rows_then); uniform priors:
        // the common factor 1/q is applied at the store
        if constexpr (KH > 0) {
          const f32x2* hp = s_head + (x & ((1u << KH) - 1u)) * (MN - E0) * kLatticeThreads;
#pragma unroll
          for (int e = 0; e < MN; e++) fo[e] = e < E0 ? Core::f2z() : hp[(e < E0 ? 0 : e - E0) * kLatticeThreads];
          Core::template run_from_then<KH + 1, Core::NNr - K, BSIDMAP_L1_GROUP>(lane, x, p, fo, add);
        } else {
          Core::template run_prefix_then<K, BSIDMAP_L1_GROUP>(lane, x, p, fo, add);
        }
      }
      Core::template apply_last_rows<K>(lane, cur, p, acc);
      if (!first) {
#pragma unroll
        for (int e = 0; e < MN; e++) acc[e] = fadd2(acc[e], res[e * kLatticeThreads]);
      }
    }
    const float sc = p.priors ? 1.f : 1.f / p.q;
    if (A.in) {
      float* out = gsum_block(p, A.f, i) + A.mi;
#pragma unroll
      for (int e = 0; e < MN; e++) out[(size_t)e * p.Mtp] = out_valid(p, A, e) ? sc * lo_of(acc[e]) : 0.f;
    }
    if (B.in) {
      float* out = gsum_block(p, B.f, i) + B.mi;
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
    if (__any_sync(0xffffffffu, alpha_live(p, false, wb, G, i))) {
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
      float* out = gsum_block(p, G.f, i) + G.mi;
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
  const double* brow = beta_row(p, G.f, i + 1);
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
  const double* brow = beta_row(p, A.f, i + 1);
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

// Lattice rows per dispatch group in the APP kernels (row pairs where the register budget allows
// 3 CTAs/SM)
#ifndef BSIDMAP_APP_GROUP
#define BSIDMAP_APP_GROUP (Core::kMinBlocks > 2 ? 2 : 1)
#endif
// the APP kernels with two folded rows: four weight tables per lane in smem
#ifndef BSIDMAP_APP_MINB_KS2
#define BSIDMAP_APP_MINB_KS2 (Core::kMinBlocks > 2 ? 3 : 2)
#endif
// per-warp staging of per-lane, per-symbol terms: [q][33] (odd stride), reduced over the lanes once
// after the symbol loop instead of one shuffle chain per symbol
__host__ __device__ __forceinline__ size_t app_stage_floats(int q) { return (size_t)q * 33; }
// Symbols are visited in lexicographic codeword order (DecodeParams::Cp, prepared at create) so
// that lattice rows 1..KP (run_head) are computed once per distinct prefix; KP = 0: natural order.
// The prefix length that saves the most nodes for random codebooks: ~log2(q) - 1.
__host__ __device__ __forceinline__ int app_prefix_bits(int q, int n) {
  int kp = q <= 8 ? 2 : q <= 16 ? 3 : 4;
  return kp <= n - 2 ? kp : 0;
}

template <class Core>
__global__ void __launch_bounds__(kLatticeThreads) k_gamma_dump_x2(const DecodeParams p) {
  using f32x2 = typename Core::P2;
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
  k.app = nullptr;
  // one folded row on the pair core: two (four smem weight tables per lane) measured slower with the
  // live-window APP (C4 pass 2 33.7 vs 23.7 ms, C2 29.4 vs 26.1; tools/exp_appkpks.sh)
  k.app_ks_auto = 1;
  k.app_live[0][0] = k_app_live_x2<typename Core::AsmCore, 0, 1>;
  k.app_live[0][1] = k_app_live_x2<typename Core::AsmCore, 2, 1>;
  k.app_live[0][2] = k_app_live_x2<typename Core::AsmCore, 3, 1>;
  k.app_live[0][3] = k_app_live_x2<typename Core::AsmCore, 4, 1>;
  k.app_live[1][0] = k_app_live_x2<typename Core::AsmCore, 0, 2>;
  k.app_live[1][1] = k_app_live_x2<typename Core::AsmCore, 2, 2>;
  k.app_live[1][2] = k_app_live_x2<typename Core::AsmCore, 3, 2>;
  k.app_live[1][3] = k_app_live_x2<typename Core::AsmCore, 4, 2>;
  k.app_live_W = 2;
  {
    using Core_ = Core;
    constexpr int minb = BSIDMAP_L1C_MINB;
    for (int K = 2; K <= 3; K++)
      k.l1_head_bytes[K - 2] = l1_head_bytes(l1_head_rows(Core_::NNr, Core_::Lo, Core_::Mn, K, minb), Core_::Lo, Core_::Mn);
  }
  k.app_stored = k_app_stored<Core::Mn>;
  k.gamma_dump = k_gamma_dump_x2<Core>;
  k.nodes = nodes;
  k.W = 2;
  k.l1_W = 2;
  k.l1_steps = true;
  k.ab_warp[0] = k_alpha_beta_warp<1, Core::Mn>;
  k.ab_warp[1] = k_alpha_beta_warp<2, Core::Mn>;
  k.ab_warp[2] = k_alpha_beta_warp<4, Core::Mn>;
  return k;
}

}  // namespace bsidmap
