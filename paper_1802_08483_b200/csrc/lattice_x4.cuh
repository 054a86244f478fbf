// lattice_x4.cuh -- the spec lattice core on FOUR consecutive windows per lane (two FP32 pairs).
//
// Same recursion as SpecCoreX2 (rescaled G = F / Pd^r, two FFMA2 per node), but a
// lane owns the windows of four consecutive start drifts m'_0 .. m'_0 + 3 of one (frame, i):
// pair A = (m'_0, m'_0 + 1), pair B = (m'_0 + 2, m'_0 + 3).  Their received windows are one
// bit stream shifted by 0..3 bits, so ONE table of Q-dot pairs
//   T_x[j'] = ((Q/Pd)(y_{s0+j'-1} | x), (Q/Pd)(y_{s0+j'} | x)),   j' = 1 .. J+2,
// serves both pairs: column j of pair A reads T_x[j], column j of pair B reads T_x[j+2].
// Per lattice row the symbol's bit x_r is warp-uniform (one branch), and the row's two
// independent insertion chains (A and B) interleave -- twice the ILP and half the branch
// and table cost per window of the two-window core.
#pragma once
#include "lattice_x2.cuh"

namespace bsidmap {

template <int NN, int LO, int MN>
struct SpecCoreX4 {
  static constexpr int Mn = MN;
  static constexpr int W = 4;
  static constexpr int J = NN + LO + MN - 1;  // last window column n + m_n^+
  static_assert(MN >= 1 && MN <= kMaxMn && LO <= 0 && LO + MN - 1 >= 0 && J + 3 <= kMaxWindow, "shape");

  struct Lane {
    f32x2 q1[J + 3];  // T_1[j'], j' = 1..J+2
    f32x2 q0[J + 3];  // T_0[j']
  };

  // win: received bits from s0 = n i + m'_0 on (bit t = y_{s0+t}; bits before the frame start are 0)
  __device__ __forceinline__ static void init(Lane& L, uint64_t win, const DecodeParams& p) {
#pragma unroll
    for (int j = 1; j <= J + 2; j++) {
      const bool ya = (win >> (j - 1)) & 1ull, yb = (win >> j) & 1ull;
      L.q1[j] = pk(ya ? p.lc.qm : p.lc.qs, yb ? p.lc.qm : p.lc.qs);
      L.q0[j] = pk(ya ? p.lc.qs : p.lc.qm, yb ? p.lc.qs : p.lc.qm);
    }
  }

  template <int R>
  __device__ __forceinline__ static void row(f32x2 (&fa)[MN], f32x2 (&fb)[MN], const f32x2 (&Q)[J + 3], f32x2 a2) {
    constexpr bool kLast = (R == NN);
    f32x2 pa = 0ull, pb = 0ull;
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const int j = R + LO + e;
      if (j < 0) continue;  // structurally zero
      f32x2 va, vb;
      if (j == 0) {
        va = fa[e + 1];  // column 0: deletions only, G_{r,0} = G_{r-1,0}
        vb = fb[e + 1];
      } else {
        const f32x2 ua = (e + 1 < MN) ? ffma2(Q[j], fa[e], fa[e + 1]) : fmul2(Q[j], fa[e]);
        const f32x2 ub = (e + 1 < MN) ? ffma2(Q[j + 2], fb[e], fb[e + 1]) : fmul2(Q[j + 2], fb[e]);
        va = (!kLast && e > 0) ? ffma2(a2, pa, ua) : ua;
        vb = (!kLast && e > 0) ? ffma2(a2, pb, ub) : ub;
      }
      fa[e] = va;
      fb[e] = vb;
      pa = va;
      pb = vb;
    }
  }

  template <int R, int RLAST>
  __device__ __forceinline__ static void rows(f32x2 (&fa)[MN], f32x2 (&fb)[MN], uint32_t x, const Lane& L, f32x2 a2) {
    if constexpr (R <= RLAST) {
      if ((x >> (R - 1)) & 1u)
        row<R>(fa, fb, L.q1, a2);
      else
        row<R>(fa, fb, L.q0, a2);
      rows<R + 1, RLAST>(fa, fb, x, L, a2);
    }
  }

  // Rows 1..n-1 of both pairs (the last row is folded into the APP weights, see last_row_weights).
  __device__ __forceinline__ static void run_penultimate(const Lane& L, uint32_t x, const DecodeParams& p,
                                                         f32x2 (&fa)[MN], f32x2 (&fb)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) fa[e] = fb[e] = pk(p.lc.row0[e], p.lc.row0[e]);
    rows<1, NN - 1>(fa, fb, x, L, pk(p.lc.a, p.lc.a));
  }

  // Rows 1..n-K and, separately, the last K rows for a codeword-suffix class (SpecCoreX2::run_prefix).
  template <int K>
  __device__ __forceinline__ static void run_prefix(const Lane& L, uint32_t x, const DecodeParams& p,
                                                    f32x2 (&fa)[MN], f32x2 (&fb)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) fa[e] = fb[e] = pk(p.lc.row0[e], p.lc.row0[e]);
    rows<1, NN - K>(fa, fb, x, L, pk(p.lc.a, p.lc.a));
  }
  template <int K>
  __device__ __forceinline__ static void apply_last_rows(const Lane& L, uint32_t cls, const DecodeParams& p,
                                                         f32x2 (&fa)[MN], f32x2 (&fb)[MN]) {
    rows<NN - K + 1, NN>(fa, fb, cls << (NN - K), L, pk(p.lc.a, p.lc.a));
  }

  // Last-row weights of one pair (SpecCoreX2::last_row_weights); kB selects pair B's columns (j + 2).
  template <bool kB, class BtAt, class W1At, class W0At>
  __device__ __forceinline__ static void last_row_weights(const Lane& L, BtAt bt, W1At w1, W0At w0) {
    constexpr int S = kB ? 2 : 0;
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const int j = NN + LO + e;
      const f32x2 del = (e >= 1) ? bt(e - 1) : 0ull;
      if (j >= 1) {
        w1(e) = ffma2(bt(e), L.q1[(j < 1 ? 1 : j) + S], del);
        w0(e) = ffma2(bt(e), L.q0[(j < 1 ? 1 : j) + S], del);
      } else {
        w1(e) = del;
        w0(e) = del;
      }
    }
  }

  static constexpr long nodes() { return (long)NN * MN - (long)LO * (LO - 1) / 2; }
};

}  // namespace bsidmap
