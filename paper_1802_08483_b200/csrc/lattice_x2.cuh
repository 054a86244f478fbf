// lattice_x2.cuh -- the spec lattice core on packed FP32 pairs (FFMA2, sm_100a).
//
// Same recursion as SpecCore (lattice.cuh: corridor nodes only, rescaled
// G = F / Pd^r so a node is u = (Q/Pd) G_{r-1,j-1} + G_{r-1,j};
// G_{r,j} = 1/2 Pi G_{r,j-1} + u), but every lane runs TWO windows -- two
// start drifts m' of the same (frame chunk, i) -- for the same symbol D, so
// x = C_i(D) and the row branch stay warp-uniform and every node of both
// lattices is one fma.rn.f32x2.  Measured on B200 (tools/ubench): a scalar
// FFMA with three register sources issues at ~0.69 of the FP32 peak, the
// packed FFMA2 with three register-pair sources at ~0.98 -- the per-lane Q-dot
// operand makes the scalar node FFMA a three-register one, the packed one
// is not penalised.
#pragma once
#include "common.cuh"

namespace bsidmap {

// A pair of FP32 values (lo = window a, hi = window b) and the sm_100 packed FP32 arithmetic
// (fma.rn.f32x2 / add.rn.f32x2 / mul.rn.f32x2), in two representations with the same results:
//  - float2 through the CUDA builtins: the compiler sees two 32-bit registers (fewer moves; pass 1
//    C3-C5 2-4 % faster than the 64-bit form, tools/gpu_quick2.sh r02 q3);
//  - one 64-bit register through inline PTX: the pair live-window APP keeps it (with float2 its C2
//    instance spills 228 B and runs 26.0 -> 29.7 ms).
// A core picks one (SpecCoreX2<..., P2T>); the kernels take the type from their core.
typedef float2 f32x2;
typedef unsigned long long u64x2;

__device__ __forceinline__ float lo_of(float2 v) { return v.x; }
__device__ __forceinline__ float hi_of(float2 v) { return v.y; }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

__device__ __forceinline__ float lo_of(u64x2 v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi_of(u64x2 v) { return __uint_as_float((unsigned)(v >> 32)); }
__device__ __forceinline__ u64x2 ffma2(u64x2 a, u64x2 b, u64x2 c) {
  u64x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64x2 fadd2(u64x2 a, u64x2 b) {
  u64x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64x2 fmul2(u64x2 a, u64x2 b) {
  u64x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

template <class P2>
__device__ __forceinline__ P2 pair_of(float lo, float hi);
template <>
__device__ __forceinline__ float2 pair_of<float2>(float lo, float hi) { return make_float2(lo, hi); }
template <>
__device__ __forceinline__ u64x2 pair_of<u64x2>(float lo, float hi) {
  return (u64x2)__float_as_uint(lo) | ((u64x2)__float_as_uint(hi) << 32);
}

template <int NN, int LO, int MN, class P2T = float2>
struct SpecCoreX2 {
  using P2 = P2T;                                       // the pair representation of this core
  using f32x2 = P2T;
  using AsmCore = SpecCoreX2<NN, LO, MN, u64x2>;        // the same core on 64-bit pairs (pair APP)
  __device__ __forceinline__ static P2 pk(float lo, float hi) { return pair_of<P2>(lo, hi); }
  __device__ __forceinline__ static P2 f2z() { return pair_of<P2>(0.f, 0.f); }
  static constexpr int Mn = MN;
  static constexpr int NNr = NN;  // lattice rows n
  static constexpr int Lo = LO;   // m_n^-
  static constexpr int W = 2;
  static constexpr int J = NN + LO + MN - 1;  // last window column n + m_n^+
  static_assert(MN >= 1 && MN <= kMaxMn && LO <= 0 && LO + MN - 1 >= 0 && J <= kMaxWindow, "shape");
  // register estimate: Q-dot tables 4J + band and accumulator 4 M_n + ~30; 3 CTAs/SM fit 168 regs
  static constexpr int kMinBlocks = (4 * J + 4 * MN + 30 <= 168) ? 3 : 2;

  struct Lane {
    f32x2 q1[J + 1];  // (Q/Pd)(y_j | x = 1) of windows (a, b), j = 1..J
    f32x2 q0[J + 1];  // (Q/Pd)(y_j | x = 0)
  };

  __device__ __forceinline__ static void init(Lane& L, uint64_t wa, uint64_t wb, const DecodeParams& p) {
#pragma unroll
    for (int j = 1; j <= J; j++) {
      const bool ya = (wa >> (j - 1)) & 1ull, yb = (wb >> (j - 1)) & 1ull;
      L.q1[j] = pk(ya ? p.lc.qm : p.lc.qs, yb ? p.lc.qm : p.lc.qs);
      L.q0[j] = pk(ya ? p.lc.qs : p.lc.qm, yb ? p.lc.qs : p.lc.qm);
    }
  }

  // Row R from row R-1 held in s into d (kInPlace: d is s; node e reads s[e], s[e+1] before d[e] is
  // written, so the update runs in place).  A separate d lets a consumer keep s (the APP's shared
  // prefix row) without copying it first.
  template <int R, bool kInPlace = true>
  __device__ __forceinline__ static void row_from(f32x2 (&d)[MN], const f32x2 (&s)[MN], const f32x2 (&Q)[J + 1],
                                                  f32x2 a2) {
    constexpr bool kLast = (R == NN);
    f32x2 prev = f2z();
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const int j = R + LO + e;
      if (j < 0) {  // structurally zero
        if constexpr (!kInPlace) d[e] = f2z();
        continue;
      }
      f32x2 v;
      if (j == 0) {
        v = s[e + 1];  // column 0: deletions only, G_{r,0} = G_{r-1,0}
      } else {
        const f32x2 u = (e + 1 < MN) ? ffma2(Q[j], s[e], s[e + 1]) : fmul2(Q[j], s[e]);
        v = (!kLast && e > 0) ? ffma2(a2, prev, u) : u;
      }
      d[e] = v;
      prev = v;
    }
  }
  template <int R>
  __device__ __forceinline__ static void row(f32x2 (&f)[MN], const f32x2 (&Q)[J + 1], f32x2 a2) {
    row_from<R, true>(f, f, Q, a2);
  }

  // Rows are issued in groups of G (1, 2 or 3): a 2^G-way branch on (x_R .. x_{R+G-1}) puts the
  // group's rows in one basic block so their insertion chains interleave (row R+1 node e needs
  // row R nodes e, e+1) and the per-row dispatch cost is paid once per group.
  template <int R, int G, int RLAST = NN>
  __device__ __forceinline__ static void rows(f32x2 (&f)[MN], uint32_t x, const Lane& L, f32x2 a2) {
    if constexpr (G >= 3 && R + 2 <= RLAST) {
      switch ((x >> (R - 1)) & 7u) {
        case 0u: row<R>(f, L.q0, a2); row<R + 1>(f, L.q0, a2); row<R + 2>(f, L.q0, a2); break;
        case 1u: row<R>(f, L.q1, a2); row<R + 1>(f, L.q0, a2); row<R + 2>(f, L.q0, a2); break;
        case 2u: row<R>(f, L.q0, a2); row<R + 1>(f, L.q1, a2); row<R + 2>(f, L.q0, a2); break;
        case 3u: row<R>(f, L.q1, a2); row<R + 1>(f, L.q1, a2); row<R + 2>(f, L.q0, a2); break;
        case 4u: row<R>(f, L.q0, a2); row<R + 1>(f, L.q0, a2); row<R + 2>(f, L.q1, a2); break;
        case 5u: row<R>(f, L.q1, a2); row<R + 1>(f, L.q0, a2); row<R + 2>(f, L.q1, a2); break;
        case 6u: row<R>(f, L.q0, a2); row<R + 1>(f, L.q1, a2); row<R + 2>(f, L.q1, a2); break;
        default: row<R>(f, L.q1, a2); row<R + 1>(f, L.q1, a2); row<R + 2>(f, L.q1, a2); break;
      }
      rows<R + 3, G, RLAST>(f, x, L, a2);
    } else if constexpr (G >= 2 && R + 1 <= RLAST) {
      switch ((x >> (R - 1)) & 3u) {
        case 0u: row<R>(f, L.q0, a2); row<R + 1>(f, L.q0, a2); break;
        case 1u: row<R>(f, L.q1, a2); row<R + 1>(f, L.q0, a2); break;
        case 2u: row<R>(f, L.q0, a2); row<R + 1>(f, L.q1, a2); break;
        default: row<R>(f, L.q1, a2); row<R + 1>(f, L.q1, a2); break;
      }
      rows<R + 2, G, RLAST>(f, x, L, a2);
    } else if constexpr (R <= RLAST) {
      if ((x >> (R - 1)) & 1u)
        row<R>(f, L.q1, a2);
      else
        row<R>(f, L.q0, a2);
      rows<R + 1, G, RLAST>(f, x, L, a2);
    }
  }

  // Rows 1..n-1 only: f[e] <- G_{n-1} in diagonal coordinates.  A consumer that only needs
  // t = sum_k bt(k) G_n(k) folds the last row (eqn:F_lastrow) into its weights:
  // t = sum_e G_{n-1}[e] w_{x_n}[e], w_x[e] = bt[e-1] + bt[e] (Q/Pd)(y_{n+k_e} | x)  (last_row_weights).
  template <int G = 1>
  __device__ __forceinline__ static void run_penultimate(const Lane& L, uint32_t x, const DecodeParams& p,
                                                         f32x2 (&f)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = pk(p.lc.row0[e], p.lc.row0[e]);
    rows<1, G, NN - 1>(f, x, L, pk(p.lc.a, p.lc.a));
  }

  // Prefix sharing (pass 2): rows 1..KP depend only on the codeword's first KP bits, so symbols
  // visited in order of those bits share them -- run_head once per distinct prefix, run_tail
  // (rows KP+1..n-1) per symbol from a copy of the head's row.  Same operations, same order:
  // bit-identical to run_penultimate.
  template <int KP, int G = 1>
  __device__ __forceinline__ static void run_head(const Lane& L, uint32_t x, const DecodeParams& p, f32x2 (&f)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = pk(p.lc.row0[e], p.lc.row0[e]);
    rows<1, G, KP>(f, x, L, pk(p.lc.a, p.lc.a));
  }
  // Rows R0..RL on f (already holding row R0 - 1), then tail(f) in the last group's basic block.
  template <int R0, int RL, int G, class Tail>
  __device__ __forceinline__ static void run_from_then(const Lane& L, uint32_t x, const DecodeParams& p,
                                                       f32x2 (&f)[MN], Tail& tail) {
    rows_then<R0, G, RL>(f, x, L, pk(p.lc.a, p.lc.a), tail);
  }
  // First node of row R that can be non-zero (nodes e with column R + m_n^- + e < 0 are structurally 0).
  static constexpr int row_e0(int R) { return (R + LO) < 0 ? -(R + LO) : 0; }
  template <int KP, int G = 1>
  __device__ __forceinline__ static void run_tail(const Lane& L, uint32_t x, const DecodeParams& p, f32x2 (&f)[MN]) {
    rows<KP + 1, G, NN - 1>(f, x, L, pk(p.lc.a, p.lc.a));
  }

  // Rows 1..n-K (the rows that depend on codeword bits other than the last K) and, separately,
  // the last K rows for the class cls = (x_{n-K+1}..x_n) applied to any vector f: the lattice rows
  // are linear in the row they read, so sum_D P(D) G_n(D) = sum_cls Last_cls(sum_{D in cls} P(D) G_{n-K}(D)).
  template <int K, int G = 1>
  __device__ __forceinline__ static void run_prefix(const Lane& L, uint32_t x, const DecodeParams& p, f32x2 (&f)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = pk(p.lc.row0[e], p.lc.row0[e]);
    rows<1, G, NN - K>(f, x, L, pk(p.lc.a, p.lc.a));
  }
  template <int K, int G, class Tail>
  __device__ __forceinline__ static void run_prefix_then(const Lane& L, uint32_t x, const DecodeParams& p,
                                                         f32x2 (&f)[MN], Tail& tail) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = pk(p.lc.row0[e], p.lc.row0[e]);
    rows_then<1, G, NN - K>(f, x, L, pk(p.lc.a, p.lc.a), tail);
  }
  template <int K>
  __device__ __forceinline__ static void apply_last_rows(const Lane& L, uint32_t cls, const DecodeParams& p,
                                                         f32x2 (&f)[MN]) {
    rows<NN - K + 1, false, NN>(f, cls << (NN - K), L, pk(p.lc.a, p.lc.a));
  }

  // rows<R, G, RLAST> followed by tail(f), with the tail placed inside each branch of the group
  // that ends at row RLAST: the consumer of the last row (the APP's weight dot) shares that basic
  // block with the row's insertion chain, so the two interleave (G <= 2).
  template <int R, int G, int RLAST, class Tail>
  __device__ __forceinline__ static void rows_then(f32x2 (&f)[MN], uint32_t x, const Lane& L, f32x2 a2, Tail& tail) {
    if constexpr (R > RLAST) {
      tail(f);
    } else if constexpr (G >= 2 && R + 1 <= RLAST) {
      constexpr bool kEnd = (R + 1 == RLAST);
      switch ((x >> (R - 1)) & 3u) {
        case 0u: row<R>(f, L.q0, a2); row<R + 1>(f, L.q0, a2); if constexpr (kEnd) tail(f); break;
        case 1u: row<R>(f, L.q1, a2); row<R + 1>(f, L.q0, a2); if constexpr (kEnd) tail(f); break;
        case 2u: row<R>(f, L.q0, a2); row<R + 1>(f, L.q1, a2); if constexpr (kEnd) tail(f); break;
        default: row<R>(f, L.q1, a2); row<R + 1>(f, L.q1, a2); if constexpr (kEnd) tail(f); break;
      }
      if constexpr (!kEnd) rows_then<R + 2, G, RLAST>(f, x, L, a2, tail);
    } else {
      constexpr bool kEnd = (R == RLAST);
      if ((x >> (R - 1)) & 1u) {
        row<R>(f, L.q1, a2);
        if constexpr (kEnd) tail(f);
      } else {
        row<R>(f, L.q0, a2);
        if constexpr (kEnd) tail(f);
      }
      if constexpr (!kEnd) rows_then<R + 1, G, RLAST>(f, x, L, a2, tail);
    }
  }

  // Rows 1..RL, and rows KP+1..RL after a shared head (the APP pass with the last n - RL rows
  // folded into its weights); the *_then forms end with tail(f) (rows_then).
  template <int RL, int G = 1>
  __device__ __forceinline__ static void run_to(const Lane& L, uint32_t x, const DecodeParams& p, f32x2 (&f)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = pk(p.lc.row0[e], p.lc.row0[e]);
    rows<1, G, RL>(f, x, L, pk(p.lc.a, p.lc.a));
  }
  template <int KP, int RL, int G = 1>
  __device__ __forceinline__ static void run_tail_to(const Lane& L, uint32_t x, const DecodeParams& p,
                                                     f32x2 (&f)[MN]) {
    rows<KP + 1, G, RL>(f, x, L, pk(p.lc.a, p.lc.a));
  }
  template <int RL, int G, class Tail>
  __device__ __forceinline__ static void run_to_then(const Lane& L, uint32_t x, const DecodeParams& p, f32x2 (&f)[MN],
                                                     Tail& tail) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = pk(p.lc.row0[e], p.lc.row0[e]);
    rows_then<1, G, RL>(f, x, L, pk(p.lc.a, p.lc.a), tail);
  }
  template <int KP, int RL, int G, class Tail>
  __device__ __forceinline__ static void run_tail_to_then(const Lane& L, uint32_t x, const DecodeParams& p,
                                                          f32x2 (&f)[MN], Tail& tail) {
    rows_then<KP + 1, G, RL>(f, x, L, pk(p.lc.a, p.lc.a), tail);
  }
  // The same from the shared prefix row fh into f: the first row group reads fh and writes f (no
  // copy of fh), the rest runs in place on f.  Same operations in the same order as copying fh to f
  // and calling run_tail_to_then (bit-identical).
  template <int KP, int RL, int G, class Tail>
  __device__ __forceinline__ static void run_tail_from_then(const Lane& L, uint32_t x, const DecodeParams& p,
                                                            const f32x2 (&fh)[MN], f32x2 (&f)[MN], Tail& tail) {
    constexpr int R = KP + 1;
    const f32x2 a2 = pk(p.lc.a, p.lc.a);
    if constexpr (R > RL) {
#pragma unroll
      for (int e = 0; e < MN; e++) f[e] = fh[e];
      tail(f);
    } else if constexpr (G >= 2 && R + 1 <= RL) {
      constexpr bool kEnd = (R + 1 == RL);
      switch ((x >> (R - 1)) & 3u) {
        case 0u: row_from<R, false>(f, fh, L.q0, a2); row<R + 1>(f, L.q0, a2); if constexpr (kEnd) tail(f); break;
        case 1u: row_from<R, false>(f, fh, L.q1, a2); row<R + 1>(f, L.q0, a2); if constexpr (kEnd) tail(f); break;
        case 2u: row_from<R, false>(f, fh, L.q0, a2); row<R + 1>(f, L.q1, a2); if constexpr (kEnd) tail(f); break;
        default: row_from<R, false>(f, fh, L.q1, a2); row<R + 1>(f, L.q1, a2); if constexpr (kEnd) tail(f); break;
      }
      if constexpr (!kEnd) rows_then<R + 2, G, RL>(f, x, L, a2, tail);
    } else {
      constexpr bool kEnd = (R == RL);
      if ((x >> (R - 1)) & 1u) {
        row_from<R, false>(f, fh, L.q1, a2);
        if constexpr (kEnd) tail(f);
      } else {
        row_from<R, false>(f, fh, L.q0, a2);
        if constexpr (kEnd) tail(f);
      }
      if constexpr (!kEnd) rows_then<R + 1, G, RL>(f, x, L, a2, tail);
    }
  }

  // Transpose of lattice row R (R < n) with Q-dot table Q: weights w on the row's outputs G_R ->
  // weights wi on its input row G_{R-1}, so that sum_e w[e] G_R[e] = sum_e wi[e] G_{R-1}[e].
  // Row R: v_e = [chain] a v_{e-1} + Q_j G_{R-1}[e] + G_{R-1}[e+1]  (j = R + m_n^- + e >= 1),
  //        v_e = G_{R-1}[e+1] (j = 0), structurally zero (j < 0); the chain runs for e > 0, j >= 1.
  // Backward: dv_e = w_e + a dv_{e+1} [chain at e+1]; wi_e = [j_e >= 1] dv_e Q_{j_e} + [j_{e-1} >= 0] dv_{e-1}.
  template <int R>
  __device__ __forceinline__ static void row_transpose(const f32x2 (&w)[MN], f32x2 (&wi)[MN], const f32x2 (&Q)[J + 1],
                                                       f32x2 a2) {
    static_assert(R < NN, "the last row is folded by last_row_weights");
    f32x2 dv[MN];
#pragma unroll
    for (int e = MN - 1; e >= 0; e--) {
      const int j = R + LO + e;
      const int jn = j + 1;  // column of node e + 1
      const bool chain_next = (e + 1 < MN) && (jn >= 1) && (e + 1 > 0);
      dv[e] = (j < 0) ? f2z() : (chain_next ? ffma2(a2, dv[e + 1 < MN ? e + 1 : e], w[e]) : w[e]);
    }
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const int j = R + LO + e;
      const f32x2 left = (e >= 1 && j - 1 >= 0) ? dv[e >= 1 ? e - 1 : 0] : f2z();
      wi[e] = (j >= 1) ? ffma2(dv[e], Q[j < 1 ? 1 : j], left) : left;
    }
  }

  // w1 (x_n = 1), w0 (x_n = 0) of run_penultimate from the corridor weights bt[e] of both windows.
  // Row n node e' (column j'): G_n[e'] = G_{n-1}[e'+1] + [j' >= 1] (Q/Pd)_{j'} G_{n-1}[e'], so the
  // coefficient of G_{n-1}[e] in sum_e' bt[e'] G_n[e'] is bt[e-1] + [j >= 1] bt[e] (Q/Pd)_j.
  template <class BtAt, class W1At, class W0At>
  __device__ __forceinline__ static void last_row_weights(const Lane& L, BtAt bt, W1At w1, W0At w0) {
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const int j = NN + LO + e;
      const f32x2 del = (e >= 1) ? bt(e - 1) : f2z();
      if constexpr (NN + LO >= 1) {  // every last-row column is >= 1
        w1(e) = ffma2(bt(e), L.q1[j], del);
        w0(e) = ffma2(bt(e), L.q0[j], del);
      } else {
        w1(e) = (j >= 1) ? ffma2(bt(e), L.q1[j < 1 ? 1 : j], del) : del;
        w0(e) = (j >= 1) ? ffma2(bt(e), L.q0[j < 1 ? 1 : j], del) : del;
      }
    }
  }

  // f[e] <- (window a, window b) lattice outputs for k = m_n^- + e (times lc.out_scale)
  // G: rows per dispatch group (more ILP, more code)
  template <int G = 1>
  __device__ __forceinline__ static void run(const Lane& L, uint32_t x, const DecodeParams& p, f32x2 (&f)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = pk(p.lc.row0[e], p.lc.row0[e]);
    rows<1, G>(f, x, L, pk(p.lc.a, p.lc.a));
  }

  static constexpr long nodes() { return (long)NN * MN - (long)LO * (LO - 1) / 2; }
};

}  // namespace bsidmap
