// lattice.cuh -- the corridor-constrained receiver-metric lattice
// as register-resident FP32 device code for sm_100a.
//
// One lattice per (frame, i, m', D) covers the largest window
// Y[n i + m' .. n(i+1) + m_n^+) and yields F_{n, n+k} for every drift change
// k in [m_n^-, m_n^+].  Only nodes inside the corridor
// m_n^- <= j - r <= m_n^+ are kept, so a lattice row is held in
// "diagonal" coordinates e = (j - r) - m_n^- in M_n registers:
//
//   F_{r,j} = 1/2 Pi F_{r,j-1} + Pd F_{r-1,j} + Q(y_j|x_r) F_{r-1,j-1}   (eqn:F, r < n)
//   F_{n,j} =                    Pd F_{n-1,j} + Q(y_j|x_n) F_{n-1,j-1}   (eqn:F_lastrow)
//
// In e-coordinates (r, j-1) is e-1, (r-1, j) is e+1 and (r-1, j-1) is e, so
// one row is new[e] = a new[e-1] + b old[e+1] + Q old[e], only the a-term on
// the serial chain.  With Pd > 0 the kernels run the exact rescaling
// G = F / Pd^r (see LatticeConst), new[e] = a new[e-1] + old[e+1] + (Q/Pd) old[e]:
// two FFMAs per node.  Writing new[e] over old[e] is safe because new[e+1]
// reads old[e+1], old[e+2] only.
//
// Lane mapping (B200 design, not the paper's): a lane owns one window
// (frame, i, m') and loops over the q symbols D.  x = C_i(D) is therefore
// warp-uniform, so "which Q-dot row" is a uniform branch on bit x_r and the
// per-lane Q-dot values Q(y_j|1), Q(y_j|0) for the window's columns are
// precomputed once per window (registers) and reused for all q lattices.
//
// Two cores: SpecCore<n, m_n^-, M_n> is fully unrolled (compile-time
// columns, structurally-zero nodes j < 0 skipped -- exactly the paper's
// node count n M_n - m_n^-(m_n^- - 1)/2); GenCore<M_n> has runtime
// n and m_n^- (rows not unrolled, Q-dot from the window bits per node).
#pragma once
#include "common.cuh"

namespace bsidmap {

// rows per dispatch group of the scalar core (2: row pairs in one 4-way branch); measured: single
// rows in the pass-1 class loop (C3 pass 1 72.3 -> 67.7 ms, C5 236 -> 228), pairs in the APP pass
// (C3 85.6 vs 87.9 ms, C5 110 vs 122) -- tools/exp_sgroup.sh
#ifndef BSIDMAP_SCALAR_GROUP
#define BSIDMAP_SCALAR_GROUP 2
#endif
#ifndef BSIDMAP_SCALAR_L1_GROUP
#define BSIDMAP_SCALAR_L1_GROUP 1
#endif

template <int NN, int LO, int MN>
struct SpecCore {
  static constexpr int Mn = MN;
  static constexpr int NNr = NN;  // lattice rows n
  static constexpr int lo = LO;
  static constexpr int hi = LO + MN - 1;
  static constexpr int J = NN + LO + MN - 1;  // last window column n + m_n^+
  static_assert(MN >= 1 && MN <= kMaxMn, "corridor width");
  static_assert(LO <= 0 && LO + MN - 1 >= 0, "corridor must contain 0");
  static_assert(J <= kMaxWindow, "window must fit 64 bits");

  struct Lane {
    float q1[J + 1];  // Q(y_j | x = 1), j = 1..J
    float q0[J + 1];  // Q(y_j | x = 0)
  };

  __device__ __forceinline__ static void init(Lane& L, uint64_t win, const DecodeParams& p) {
#pragma unroll
    for (int j = 1; j <= J; j++) {
      const bool y = (win >> (j - 1)) & 1ull;
      L.q1[j] = y ? p.lc.qm : p.lc.qs;
      L.q0[j] = y ? p.lc.qs : p.lc.qm;
    }
  }

  // Row R from row R-1 held in s into d (kInPlace: d is s, see SpecCoreX2::row_from).
  template <int R, bool kRescaled, bool kInPlace = true>
  __device__ __forceinline__ static void row_from(float (&d)[MN], const float (&s)[MN], const float (&Q)[J + 1],
                                                  const LatticeConst& lc) {
    constexpr bool kLast = (R == NN);
    float prev = 0.f;
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const int j = R + LO + e;  // lattice column of this node
      if (j < 0) {               // left of column 0: structurally zero, stays 0
        if constexpr (!kInPlace) d[e] = 0.f;
        continue;
      }
      float v;
      if (j == 0) {
        // column 0 is reached by deletions only: F_{r,0} = Pd F_{r-1,0}, i.e. G_{r,0} = G_{r-1,0}
        v = kRescaled ? s[e + 1] : lc.b * s[e + 1];
      } else {
        float u;
        if (e + 1 < MN)  // deletion Pd F_{r-1,j} + transmission Q F_{r-1,j-1}
          u = kRescaled ? fmaf(Q[j], s[e], s[e + 1]) : fmaf(Q[j], s[e], lc.b * s[e + 1]);
        else
          u = Q[j] * s[e];
        v = (!kLast && e > 0) ? fmaf(lc.a, prev, u) : u;  // insertion 1/2 Pi F_{r,j-1}
      }
      d[e] = v;
      prev = v;
    }
  }
  template <int R, bool kRescaled>
  __device__ __forceinline__ static void row(float (&f)[MN], const float (&Q)[J + 1], const LatticeConst& lc) {
    row_from<R, kRescaled, true>(f, f, Q, lc);
  }

  // Rows are issued in pairs: a 4-way branch on (x_R, x_{R+1}) puts rows R and R+1
  // in one basic block, so the scheduler interleaves their two insertion chains
  // (row R+1 node e only needs row R nodes e, e+1) -- ILP 2 without extra registers.
  template <int R, int RLAST = NN, int G = BSIDMAP_SCALAR_GROUP>
  __device__ __forceinline__ static void rows(float (&f)[MN], uint32_t x, const Lane& L, const LatticeConst& lc) {
    if constexpr (G >= 2 && R + 1 <= RLAST) {
      switch ((x >> (R - 1)) & 3u) {
        case 0u: row<R, true>(f, L.q0, lc); row<R + 1, true>(f, L.q0, lc); break;
        case 1u: row<R, true>(f, L.q1, lc); row<R + 1, true>(f, L.q0, lc); break;
        case 2u: row<R, true>(f, L.q0, lc); row<R + 1, true>(f, L.q1, lc); break;
        default: row<R, true>(f, L.q1, lc); row<R + 1, true>(f, L.q1, lc); break;
      }
      rows<R + 2, RLAST, G>(f, x, L, lc);
    } else if constexpr (R <= RLAST) {
      if ((x >> (R - 1)) & 1u)
        row<R, true>(f, L.q1, lc);
      else
        row<R, true>(f, L.q0, lc);
      rows<R + 1, RLAST, G>(f, x, L, lc);
    }
  }

  // rows<R, RLAST> then tail(f) inside the basic block of the last row (SpecCoreX2::rows_then)
  template <int R, int RLAST, class Tail, int G = BSIDMAP_SCALAR_GROUP>
  __device__ __forceinline__ static void rows_then(float (&f)[MN], uint32_t x, const Lane& L, const LatticeConst& lc,
                                                   Tail& tail) {
    if constexpr (R > RLAST) {
      tail(f);
    } else if constexpr (G >= 2 && R + 1 <= RLAST) {
      constexpr bool kEnd = (R + 1 == RLAST);
      switch ((x >> (R - 1)) & 3u) {
        case 0u: row<R, true>(f, L.q0, lc); row<R + 1, true>(f, L.q0, lc); if constexpr (kEnd) tail(f); break;
        case 1u: row<R, true>(f, L.q1, lc); row<R + 1, true>(f, L.q0, lc); if constexpr (kEnd) tail(f); break;
        case 2u: row<R, true>(f, L.q0, lc); row<R + 1, true>(f, L.q1, lc); if constexpr (kEnd) tail(f); break;
        default: row<R, true>(f, L.q1, lc); row<R + 1, true>(f, L.q1, lc); if constexpr (kEnd) tail(f); break;
      }
      if constexpr (!kEnd) rows_then<R + 2, RLAST, Tail, G>(f, x, L, lc, tail);
    } else {
      constexpr bool kEnd = (R == RLAST);
      if ((x >> (R - 1)) & 1u) {
        row<R, true>(f, L.q1, lc);
        if constexpr (kEnd) tail(f);
      } else {
        row<R, true>(f, L.q0, lc);
        if constexpr (kEnd) tail(f);
      }
      if constexpr (!kEnd) rows_then<R + 1, RLAST, Tail, G>(f, x, L, lc, tail);
    }
  }

  // Rows 1..n-K and the last K rows for a class (see SpecCoreX2::run_prefix / apply_last_rows).
  template <int K>
  __device__ __forceinline__ static void run_prefix(const Lane& L, uint32_t x, const DecodeParams& p, float (&f)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = p.lc.row0[e];
    if constexpr (NN - K >= 1) rows<1, NN - K, BSIDMAP_SCALAR_L1_GROUP>(f, x, L, p.lc);
  }
  template <int K>
  __device__ __forceinline__ static void apply_last_rows(const Lane& L, uint32_t cls, const DecodeParams& p,
                                                         float (&f)[MN]) {
    rows<NN - K + 1, NN, BSIDMAP_SCALAR_L1_GROUP>(f, cls << (NN - K), L, p.lc);
  }

  // Rows 1..KP (shared by symbols with the same first KP codeword bits) and rows KP+1..n-1
  // (see SpecCoreX2::run_head / run_tail).
  template <int KP>
  __device__ __forceinline__ static void run_head(const Lane& L, uint32_t x, const DecodeParams& p, float (&f)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = p.lc.row0[e];
    rows<1, KP>(f, x, L, p.lc);
  }
  template <int KP>
  __device__ __forceinline__ static void run_tail(const Lane& L, uint32_t x, const DecodeParams& p, float (&f)[MN]) {
    if constexpr (KP + 1 <= NN - 1) rows<KP + 1, NN - 1>(f, x, L, p.lc);
  }

  // Rows 1..RL, and rows KP+1..RL after a shared head (SpecCoreX2::run_to / run_tail_to).
  template <int RL>
  __device__ __forceinline__ static void run_to(const Lane& L, uint32_t x, const DecodeParams& p, float (&f)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = p.lc.row0[e];
    if constexpr (RL >= 1) rows<1, RL>(f, x, L, p.lc);
  }
  template <int KP, int RL>
  __device__ __forceinline__ static void run_tail_to(const Lane& L, uint32_t x, const DecodeParams& p, float (&f)[MN]) {
    if constexpr (KP + 1 <= RL) rows<KP + 1, RL>(f, x, L, p.lc);
  }
  template <int RL, class Tail>
  __device__ __forceinline__ static void run_to_then(const Lane& L, uint32_t x, const DecodeParams& p, float (&f)[MN],
                                                     Tail& tail) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = p.lc.row0[e];
    rows_then<1, RL>(f, x, L, p.lc, tail);
  }
  template <int KP, int RL, class Tail>
  __device__ __forceinline__ static void run_tail_to_then(const Lane& L, uint32_t x, const DecodeParams& p,
                                                          float (&f)[MN], Tail& tail) {
    rows_then<KP + 1, RL>(f, x, L, p.lc, tail);
  }
  // Rows KP+1..RL from the shared prefix row fh into f, then tail(f) in the last group's basic block
  // (kTail; else no tail): the first group reads fh and writes f, so fh is not copied first.  Same
  // operations in the same order as copying fh to f and calling run_tail_to(_then) (bit-identical).
  template <int KP, int RL, bool kTail, class Tail>
  __device__ __forceinline__ static void run_tail_from(const Lane& L, uint32_t x, const DecodeParams& p,
                                                       const float (&fh)[MN], float (&f)[MN], Tail& tail) {
    constexpr int R = KP + 1;
    constexpr int G = BSIDMAP_SCALAR_GROUP;
    const LatticeConst& lc = p.lc;
    if constexpr (R > RL) {
#pragma unroll
      for (int e = 0; e < MN; e++) f[e] = fh[e];
      if constexpr (kTail) tail(f);
    } else if constexpr (G >= 2 && R + 1 <= RL) {
      constexpr bool kEnd = kTail && (R + 1 == RL);
      switch ((x >> (R - 1)) & 3u) {
        case 0u: row_from<R, true, false>(f, fh, L.q0, lc); row<R + 1, true>(f, L.q0, lc); if constexpr (kEnd) tail(f); break;
        case 1u: row_from<R, true, false>(f, fh, L.q1, lc); row<R + 1, true>(f, L.q0, lc); if constexpr (kEnd) tail(f); break;
        case 2u: row_from<R, true, false>(f, fh, L.q0, lc); row<R + 1, true>(f, L.q1, lc); if constexpr (kEnd) tail(f); break;
        default: row_from<R, true, false>(f, fh, L.q1, lc); row<R + 1, true>(f, L.q1, lc); if constexpr (kEnd) tail(f); break;
      }
      if constexpr (R + 2 <= RL) {
        if constexpr (kTail) rows_then<R + 2, RL>(f, x, L, lc, tail);
        else rows<R + 2, RL>(f, x, L, lc);
      }
    } else {
      constexpr bool kEnd = kTail && (R == RL);
      if ((x >> (R - 1)) & 1u) {
        row_from<R, true, false>(f, fh, L.q1, lc);
        if constexpr (kEnd) tail(f);
      } else {
        row_from<R, true, false>(f, fh, L.q0, lc);
        if constexpr (kEnd) tail(f);
      }
      if constexpr (R + 1 <= RL) {
        if constexpr (kTail) rows_then<R + 1, RL>(f, x, L, lc, tail);
        else rows<R + 1, RL>(f, x, L, lc);
      }
    }
  }
  // Transpose of lattice row R < n (SpecCoreX2::row_transpose): weights on G_R -> weights on G_{R-1}.
  template <int R>
  __device__ __forceinline__ static void row_transpose(const float (&w)[MN], float (&wi)[MN], const float (&Q)[J + 1],
                                                       float a) {
    static_assert(R < NN, "the last row is folded by last_row_weights");
    float dv[MN];
#pragma unroll
    for (int e = MN - 1; e >= 0; e--) {
      const int j = R + LO + e;
      const bool chain_next = (e + 1 < MN) && (j + 1 >= 1);
      dv[e] = (j < 0) ? 0.f : (chain_next ? fmaf(a, dv[e + 1 < MN ? e + 1 : e], w[e]) : w[e]);
    }
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const int j = R + LO + e;
      const float left = (e >= 1 && j - 1 >= 0) ? dv[e >= 1 ? e - 1 : 0] : 0.f;
      wi[e] = (j >= 1) ? fmaf(dv[e], Q[j < 1 ? 1 : j], left) : left;
    }
  }

  // Rows 1..n-1 only (see SpecCoreX2::run_penultimate / last_row_weights).
  __device__ __forceinline__ static void run_penultimate(const Lane& L, uint32_t x, const DecodeParams& p,
                                                         float (&f)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = p.lc.row0[e];
    if constexpr (NN >= 2) rows<1, NN - 1>(f, x, L, p.lc);
  }
  // w_x[e] = bt[e-1] + [j >= 1] bt[e] (Q/Pd)_j(x), the last row (eqn:F_lastrow) folded into t's weights.
  __device__ __forceinline__ static void last_row_weights(const Lane& L, const float (&bt)[MN], float (&w1)[MN],
                                                          float (&w0)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) {
      const int j = NN + LO + e;
      const float del = (e >= 1) ? bt[e - 1] : 0.f;
      w1[e] = (j >= 1) ? fmaf(bt[e], L.q1[j < 1 ? 1 : j], del) : del;
      w0[e] = (j >= 1) ? fmaf(bt[e], L.q0[j < 1 ? 1 : j], del) : del;
    }
  }

  // f[e] <- lattice output for drift change k = m_n^- + e (true metric = lc.out_scale * f[e]).
  // Spec cores run the rescaled recursion only (Pd > 0; the planner routes Pd = 0 to GenCore).
  __device__ __forceinline__ static void run(const Lane& L, uint32_t x, const DecodeParams& p, float (&f)[MN]) {
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = p.lc.row0[e];  // F_{0,j}: host zeroes j < 0
    rows<1>(f, x, L, p.lc);
  }

  static constexpr long nodes() {  // corridor nodes per lattice
    return (long)NN * MN - (long)LO * (LO - 1) / 2;
  }
};

template <int MN>
struct GenCore {
  static constexpr int Mn = MN;
  struct Lane {
    uint64_t win;
  };
  __device__ __forceinline__ static void init(Lane& L, uint64_t win, const DecodeParams&) { L.win = win; }

  __device__ __forceinline__ static void run(const Lane& L, uint32_t x, const DecodeParams& p, float (&f)[MN]) {
    const LatticeConst& lc = p.lc;
#pragma unroll
    for (int e = 0; e < MN; e++) f[e] = lc.row0[e];
    const int n = p.n;
    for (int r = 1; r <= n; r++) {
      const bool last = (r == n);
      const uint32_t xr = (x >> (r - 1)) & 1u;
      const int j0 = r + p.mn_lo;
      float prev = 0.f;
#pragma unroll
      for (int e = 0; e < MN; e++) {
        const int j = j0 + e;
        float v = 0.f;
        if (j >= 0) {
          float u = (e + 1 < MN) ? (lc.rescaled ? f[e + 1] : lc.b * f[e + 1]) : 0.f;
          if (j >= 1) {
            const uint32_t yb = (uint32_t)(L.win >> (j - 1)) & 1u;
            u = fmaf((yb == xr) ? lc.qm : lc.qs, f[e], u);
            if (!last && e > 0) u = fmaf(lc.a, prev, u);
          }
          v = u;
        }
        f[e] = v;
        prev = v;
      }
    }
  }
};

}  // namespace bsidmap
