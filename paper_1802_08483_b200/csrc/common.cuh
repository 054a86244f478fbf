// common.cuh -- parameters shared by the bsidmap kernels (sm_100a).
//
// Notation follows arXiv 1802.08483 (P:n = PAPER.md line n): q, n, N,
// drift limits m_n^-/m_n^+ (corridor, M_n) and m_tau^-/m_tau^+ (trellis
// states, M_tau), channel Pi, Pd, Ps.
#pragma once
#ifdef __CUDACC_RTC__  // run-time compiled shapes (jit.cu, NVRTC): no host headers
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned long size_t;
#else
#include <cstdint>
#include <cuda_runtime.h>
#endif

namespace bsidmap {

constexpr int kMaxMn = 32;        // corridor width held in registers
constexpr int kMaxWindow = 64;    // n + m_n^+ received bits per lattice window
constexpr int kLatticeSeedMaxLog2 = 80;  // F_{0,0} = 2^s, s <= 80: exact range extension of the FP32 lattice

enum FrameStatus : int32_t { kFrameOk = 0, kFrameDriftOutOfRange = 1, kFrameUnderflow = 2 };

// Channel constants of the FP32 lattice (eqn:F, eqn:F_lastrow, Q-dot P:207-215).
//
// rescaled = 1 (Pd > 0): the kernels run G_{r,j} = F_{r,j} / Pd^r, an exact
// rescaling under which eqn:F becomes
//     G_{r,j} = 1/2 Pi G_{r,j-1} + G_{r-1,j} + (Q/Pd) G_{r-1,j-1}
// -- two FFMAs per node instead of FMUL + 2 FFMA.  Every lattice output then
// carries the same factor Pd^-n 2^s, which cancels in the alpha/beta and APP
// normalisations; out_scale undoes it for debug dumps.
struct LatticeConst {
  float a;                 // 1/2 Pi   (insertion of a matching random bit)
  float b;                 // Pd       (deletion; 1 when rescaled)
  float qm;                // Pt (1 - Ps)  Q-dot for y == x   (divided by Pd when rescaled)
  float qs;                // Pt Ps        Q-dot for y != x   (divided by Pd when rescaled)
  int rescaled;            // 1: G = F / Pd^r recursion, 0: plain eqn:F
  int seed_log2;           // F_{0,0} = 2^seed_log2
  double out_scale;        // true metric = out_scale * lattice output
  float row0[kMaxMn];      // row 0 of the lattice, F_{0,j} = 2^s (1/2 Pi)^j, indexed by e = j - m_n^-
};

// Everything one decode launch needs, passed by value (lives in the constant bank).
struct DecodeParams {
  int q, n, N;
  int mn_lo, mn_hi, Mn;
  int mt_lo, mt_hi, Mt;
  int Mtp;                    // row stride of Gsum: M_tau rounded up to a multiple of 4 (16-byte rows for TMA)
  int F;                      // frames in this chunk
  const uint32_t* C;          // [N][q] codebook, decoder-owned (bit t = t-th transmitted bit)
  // Symbol visiting orders of C_i, prepared once at create (decoder-owned, [N][q]):
  const uint32_t* Cp;         // codewords in lexicographic order of (x_1, x_2, ..): every prefix group contiguous
  const uint16_t* Dp;         //   their symbols D
  const uint32_t* Cs[2];      // codewords grouped by the class of their last K = 2, 3 bits (stable)
  const uint16_t* Ds[2];      //   their symbols D
  const int* Cst[2];          //   [N][2^K + 1] first position of each class (last entry q)
  const uint32_t* rx;         // packed received words, caller-owned
  const int64_t* rx_off;      // [F] word offset of each frame in rx
  const int32_t* rho;         // [F] received length
  const float* priors;        // [F][N][q] or nullptr (uniform 1/q)
  const double* alpha0;       // [F][M_tau] frame-boundary prior alpha_0 or nullptr (= delta(0))
  const double* betaN;        // [F][M_tau] frame-boundary prior beta_N or nullptr (= delta(rho - tau))
  int32_t* status;            // [F]
  float* Gsum;                // [F][N][M_n][Mtp]  Gamma_i(m', k) = sum_D gamma_i(m', m'+k, D) (lattice scale)
  float* gamma;               // stored variant: [F][N][q][M_n][M_tau] gamma, scaled 2^80
  double* alpha;              // [F][N+1][M_tau] normalised alpha rows
  double* beta;               // [F][N+1][M_tau] normalised beta rows
  double* Lacc;               // [F][N][q] un-normalised APP accumulators
  int2* live;                 // [F][N] live windows of each APP row: (first state index, count rounded up to even)
  double live_eps;            // window (i, m') is live iff alpha_i(m') beta_i(m') > live_eps sum_m alpha_i beta_i
  int app_G;                  // frames per warp of the live-window APP kernels
  float* L;                   // [F][N][q] output APP, rows sum to 1
  double* dbg_gamma;          // debug dump [F][M_tau][M_n][q] (true scale) or nullptr
  int dbg_i;                  // symbol index of the debug dump
  int i_base;                 // first symbol index of this launch (blockIdx.y offset)
  int i_end;                  // one past the last symbol index of this launch (multi-step kernels)
  int i_steps;                // symbol indices per CTA of the multi-step kernels
  // Gamma slab (the blocked memory-reduced schedule keeps Gamma_i only for a slab of symbol
  // indices [gs_i0, gs_i0 + gs_N)): Gamma_i of frame f is block f gs_N + (i - gs_i0) of Gsum.
  // The Gamma-sum schedule keeps every block: gs_N = N, gs_i0 = 0.
  int gs_N, gs_i0;
  int askip;                  // pass 1: only windows with alpha_i(m') != 0 (recomputed Gamma, slab bwd sweep)
  // alpha/beta launches over part of the recursion: steps [ab_r0, ab_r1) (step s is symbol index s
  // forward, N - 1 - s backward), directions ab_dir (-1: both, 0: alpha only, 1: beta only); a
  // range that does not start at step 0 resumes from the stored, normalised row
  int ab_r0, ab_r1, ab_dir;
  int beta_rows;              // beta rows kept per frame: N + 1, or a ring of 3 slabs (row i at i % beta_rows)
  int2* spack;                // slab backward sweep: packed alpha-support windows per symbol-index group
  int* spack_blk;             //   its per-block scan totals (k_support_pack1/2)
  LatticeConst lc;
};

// beta_i of frame f (the whole recursion, or the slab schedule's ring of three slabs of rows).
__device__ __forceinline__ double* beta_row(const DecodeParams& p, int f, int i) {
  const int r = i < p.beta_rows ? i : i % p.beta_rows;  // no division for the whole recursion (k_live: 0.5 ms)
  return p.beta + ((size_t)f * p.beta_rows + (size_t)r) * p.Mt;
}
// (frame, i) of row `row` of a launch over symbol indices [i_base, i_base + ni) (32-bit division
// where the row count allows: the per-row kernels are short)
__device__ __forceinline__ void row_fi(long row, int ni, int i_base, int* f, int* i) {
  if (row < 0x7fffffffL) {
    const unsigned r = (unsigned)row, q = r / (unsigned)ni;
    *f = (int)q;
    *i = i_base + (int)(r - q * (unsigned)ni);
  } else {
    *f = (int)(row / ni);
    *i = i_base + (int)(row - (long)*f * ni);
  }
}

// Gamma_i block of frame f (M_n x Mtp floats) in the Gamma-sum array or the current slab.
__device__ __forceinline__ float* gsum_block(const DecodeParams& p, int f, int i) {
  return p.Gsum + ((size_t)f * p.gs_N + (i - p.gs_i0)) * p.Mn * p.Mtp;
}

// Row stride of Gsum: M_tau rounded up to whole 32-byte sectors (8 floats): every Gamma row starts a
// sector (and is a 16-byte multiple, as the TMA bulk copies of the alpha/beta kernels need).  Zeroing
// the padding in pass 1 as well (no partially written sectors, whose eviction costs a DRAM read of
// the rest: C2 2.9 GB per step) measured slower: C2 pass 1 45.7 -> 51.4 ms (more spills in the
// compute-bound loop); the reads cost no time there (DRAM at 7 % of peak).
__host__ __device__ __forceinline__ int gsum_stride(int Mt) { return (Mt + 7) & ~7; }

// Boundary row of frame f at state index m: alpha_0 (fwd) / beta_N (bwd), point masses by default.
__device__ __forceinline__ double boundary_row(const DecodeParams& p, int f, int m, bool fwd) {
  if (m >= p.Mt) return 0.0;
  if (fwd) return p.alpha0 ? p.alpha0[(size_t)f * p.Mt + m] : (m == -p.mt_lo ? 1.0 : 0.0);
  return p.betaN ? p.betaN[(size_t)f * p.Mt + m] : (m == p.rho[f] - p.n * p.N - p.mt_lo ? 1.0 : 0.0);
}

// 64 received bits starting at bit `s` of frame f (LSB-first); bits at or
// beyond rho read as 0 (they only feed lattice columns that are masked).
__device__ __forceinline__ uint64_t load_window(const DecodeParams& p, int f, int s, int rho) {
  const uint32_t* w = p.rx + p.rx_off[f];
  const int nwords = (rho + 31) >> 5;
  const int w0 = s >> 5, sh = s & 31;
  const uint32_t a = (w0 < nwords) ? __ldg(w + w0) : 0u;
  const uint32_t b = (w0 + 1 < nwords) ? __ldg(w + w0 + 1) : 0u;
  const uint32_t c = (w0 + 2 < nwords) ? __ldg(w + w0 + 2) : 0u;
  const uint32_t lo = __funnelshift_r(a, b, sh);
  const uint32_t hi = __funnelshift_r(b, c, sh);
  return (uint64_t)lo | ((uint64_t)hi << 32);
}

// Frame-constant part of a window's geometry (the lattice kernels that walk several symbol
// indices i for the same windows load it once) and the raw received words of a window.
struct WinBase {
  int f, mi, mp, rho, nwords;
  bool in, ok;
  const uint32_t* w;
};
__device__ __forceinline__ WinBase win_base(const DecodeParams& p, long g) {
  WinBase b;
  b.in = g < (long)p.F * p.Mt;
  b.f = b.in ? (int)(g / p.Mt) : 0;
  b.mi = b.in ? (int)(g - (long)b.f * p.Mt) : 0;
  b.mp = p.mt_lo + b.mi;
  b.rho = b.in ? p.rho[b.f] : 0;
  b.ok = b.in && p.status[b.f] == kFrameOk;
  b.w = p.rx + (b.in ? p.rx_off[b.f] : 0);
  b.nwords = (b.rho + 31) >> 5;
  return b;
}

// The slab schedule's backward sweep (p.askip): the windows with alpha != 0 are packed across frames.
// For symbol-index group g (the i_steps indices of one pass-1 CTA row), p.spack[g][f] = (offset of
// frame f's windows in the packed list, first window lo_f) and p.spack[g][F].x = total T; frame f
// contributes the windows [lo_f, hi_f] holding every alpha_i(m') != 0 of the group (k_support_pack*).
// Slots [0, T) are these windows (the largest f whose offset is <= slot); slots [T, F M_tau) are the
// other windows in frame order (frame f's start at f M_tau - offset_f), which only write their Gamma
// rows as 0.
__device__ __forceinline__ WinBase win_base_packed(const DecodeParams& p, long slot, int g) {
  const int2* pk = p.spack + (size_t)g * (p.F + 1);
  const long T = pk[p.F].x, Mt = p.Mt;
  WinBase b;
  b.in = slot < (long)p.F * Mt;
  const bool live = slot < T;
  const long d = live ? slot : slot - T;  // index in the live or the dead list
  int f = 0;
  if (b.in) {
    int lo = 0, hi = p.F - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      const long start = live ? (long)pk[mid].x : (long)mid * Mt - pk[mid].x;
      if (start <= d) lo = mid; else hi = mid - 1;
    }
    f = lo;
  }
  const int2 e = pk[f];
  const long start = live ? (long)e.x : (long)f * Mt - e.x;
  const int idx = (int)(d - start);
  const int w = (f + 1 < p.F ? pk[f + 1].x : (int)T) - e.x;  // frame f's live windows
  b.f = f;
  b.mi = !b.in ? 0 : live ? e.y + idx : (idx < e.y ? idx : idx + w);
  b.mp = p.mt_lo + b.mi;
  b.rho = b.in ? p.rho[f] : 0;
  b.ok = b.in && live && p.status[f] == kFrameOk;  // dead windows: Gamma rows written as 0
  b.w = p.rx + (b.in ? p.rx_off[f] : 0);
  b.nwords = (b.rho + 31) >> 5;
  return b;
}
struct Win3 {
  uint32_t a, b, c;
};
// the three words holding bits s .. s+63 (0 past the frame end; s < 0 reads from 0: inactive windows)
__device__ __forceinline__ Win3 win_words(const WinBase& b, int s) {
  const int w0 = max(s, 0) >> 5;
  Win3 r;
  r.a = (w0 < b.nwords) ? __ldg(b.w + w0) : 0u;
  r.b = (w0 + 1 < b.nwords) ? __ldg(b.w + w0 + 1) : 0u;
  r.c = (w0 + 2 < b.nwords) ? __ldg(b.w + w0 + 2) : 0u;
  return r;
}
__device__ __forceinline__ uint64_t win_bits(const Win3& r, int s) {
  const int sh = max(s, 0) & 31;
  return (uint64_t)__funnelshift_r(r.a, r.b, sh) | ((uint64_t)__funnelshift_r(r.b, r.c, sh) << 32);
}

}  // namespace bsidmap
