// k_lattice.cuh -- lattice-pass kernels, templated on the lattice core.
//
//   k_gamma_sum : a1 (step 1) -- gamma_i(m', m'+k, D) = P(D_i=D) 2^80 F_{n,n+k}
//                 (eqn:gamma P:156-161), folded over D on the fly into
//                 Gamma_i(m', k) = sum_D gamma_i (the only thing the alpha
//                 and beta recursions eqn:alpha/eqn:beta need).  Stored
//                 variant: also writes every gamma.
//   k_app       : a4 (step 3) -- recomputes gamma_i (second lattice pass,
//                 the paper's "computed at least twice") and
//                 forms sum_{m',m} alpha_i(m') gamma_i(m',m,D) beta_{i+1}(m)
//                 (eqn:L/eqn:sigma) into FP64 accumulators.
//   k_app_stored: a4 for the stored variant -- streams gamma from HBM.
//   k_gamma_dump: debug -- gamma for one i in FP64 at true scale.
//
// Grid: blockIdx.y = symbol index i (+ p.i_base), x over the flat lane index
// g = f M_tau + (m' - m_tau^-) of the chunk's frames; one lane = one window.
#pragma once
#ifndef __CUDACC_RTC__
#include <string>
#endif
#include "lattice.cuh"
#include "lattice_x2.cuh"
#include "k_alphabeta_warp.cuh"

namespace bsidmap {

constexpr int kLatticeThreads = 128;
#ifndef BSIDMAP_LATTICE_MIN_BLOCKS
#define BSIDMAP_LATTICE_MIN_BLOCKS 4
#endif
constexpr int kLatticeMinBlocks = BSIDMAP_LATTICE_MIN_BLOCKS;  // resident CTAs per SM the register budget must allow

struct LaneGeom {
  int f, mi, mp, s, rho;
  bool in, active;
  uint32_t vmask;  // bit e set iff output k = m_n^- + e is kept (see out_valid)
};

// Output k = m_n^- + e is kept iff the window is active, n + k >= 0, the window end
// n(i+1) + m = s + n + k <= rho, and m = m' + k is a trellis state (reading R5):
// an interval of e, turned into a bit mask once per window.
__device__ __forceinline__ uint32_t valid_mask(const DecodeParams& p, const LaneGeom& G) {
  const int e_lo = max(max(0, -p.n - p.mn_lo), p.mt_lo - G.mp - p.mn_lo);
  const int e_hi = min(min(p.Mn - 1, G.rho - G.s - p.n - p.mn_lo), p.mt_hi - G.mp - p.mn_lo);
  if (!G.active || e_hi < e_lo) return 0u;
  return ((2u << e_hi) - 1u) & ~((1u << e_lo) - 1u);
}

__device__ __forceinline__ LaneGeom lane_geom_at(const DecodeParams& p, int i, long g) {
  LaneGeom G;
  G.in = g < (long)p.F * p.Mt;
  G.f = G.in ? (int)(g / p.Mt) : 0;
  G.mi = G.in ? (int)(g - (long)G.f * p.Mt) : 0;
  G.mp = p.mt_lo + G.mi;                 // start drift m'
  G.s = p.n * i + G.mp;                  // window start n i + m' (eqn:gamma)
  G.rho = G.in ? p.rho[G.f] : 0;
  G.active = G.in && p.status[G.f] == kFrameOk && G.s >= 0 && G.s <= G.rho;
  G.vmask = valid_mask(p, G);
  return G;
}

__device__ __forceinline__ LaneGeom lane_geom(const DecodeParams& p, int i) {
  return lane_geom_at(p, i, (long)blockIdx.x * blockDim.x + threadIdx.x);
}

__device__ __forceinline__ bool out_valid(const DecodeParams&, const LaneGeom& G, int e) {
  return (G.vmask >> e) & 1u;
}


template <class Core, bool kStoreGamma>
__global__ void __launch_bounds__(kLatticeThreads, kLatticeMinBlocks) k_gamma_sum(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  extern __shared__ uint32_t s_C[];  // C_i(0..q-1)
  const int i = blockIdx.y + p.i_base;
  for (int t = threadIdx.x; t < p.q; t += blockDim.x) s_C[t] = p.C[(size_t)i * p.q + t];
  __syncthreads();

  const LaneGeom G = lane_geom(p, i);
  float acc[MN];
#pragma unroll
  for (int e = 0; e < MN; e++) acc[e] = 0.f;

  if (__any_sync(0xffffffffu, G.active)) {
    typename Core::Lane lane;
    Core::init(lane, G.active ? load_window(p, G.f, G.s, G.rho) : 0ull, p);
    const float* pri = p.priors ? p.priors + ((size_t)G.f * p.N + i) * p.q : nullptr;
    float* gout = kStoreGamma ? p.gamma + (((size_t)G.f * p.N + i) * p.q) * MN * p.Mt + G.mi : nullptr;
    for (int D = 0; D < p.q; D++) {
      const float P = pri ? __ldg(pri + D) : 1.f;
      float fo[MN];
      Core::run(lane, s_C[D], p, fo);
#pragma unroll
      for (int e = 0; e < MN; e++) acc[e] = fmaf(P, fo[e], acc[e]);
      if constexpr (kStoreGamma) {
        if (G.in) {
          const float sc = pri ? P : 1.f / p.q;
#pragma unroll
          for (int e = 0; e < MN; e++)
            __stcs(gout + ((size_t)D * MN + e) * p.Mt, out_valid(p, G, e) ? sc * fo[e] : 0.f);
        }
      }
    }
  } else if constexpr (kStoreGamma) {
    if (G.in) {
      float* gout = p.gamma + (((size_t)G.f * p.N + i) * p.q) * MN * p.Mt + G.mi;
      for (int D = 0; D < p.q; D++)
#pragma unroll
        for (int e = 0; e < MN; e++) __stcs(gout + ((size_t)D * MN + e) * p.Mt, 0.f);
    }
  }
  if (G.in) {
    const float sc = p.priors ? 1.f : 1.f / p.q;
    float* out = gsum_block(p, G.f, i) + G.mi;
#pragma unroll
    for (int e = 0; e < MN; e++) out[(size_t)e * p.Mtp] = out_valid(p, G, e) ? sc * acc[e] : 0.f;
  }
}

constexpr int kAppDChunk = 64;  // symbols per smem staging round of the APP passes

constexpr int kAppSegCap = 8;  // frame segments per CTA combined in shared memory before the global atomics

__host__ __device__ __forceinline__ int app_tstride(int q) { return (q < kAppDChunk ? q : kAppDChunk) + 1; }

// Segmented (per frame) reduction of the CTA's contributions w(l) * t(l, D) into
// the FP64 accumulators Lacc[f][i][D], D in [D0, D0 + nD).  s_t[l * ts + d] holds
// window l's t for symbol D0 + d (odd stride ts: conflict-free).  Level 1: every
// thread sums a contiguous chunk of 16 windows for one d, splitting at frame
// boundaries, into s_part (FP64 smem atomics); level 2: one global atomic per
// (frame segment, d).  Contains __syncthreads: every thread of the CTA calls it.
__device__ __forceinline__ void app_reduce(const DecodeParams& p, int i, int D0, int nD, const double* s_w,
                                           const float* s_t, int ts, long g0, int nwin, double* s_part) {
  constexpr int CH = 16;
  const long gend = min(g0 + (long)nwin, (long)p.F * p.Mt);
  if (g0 >= gend) return;  // uniform over the CTA
  const int nvalid = (int)(gend - g0);
  const int f0 = (int)(g0 / p.Mt), f1 = (int)((gend - 1) / p.Mt);
  const int nseg = f1 - f0 + 1;
  const bool use_smem = nseg <= kAppSegCap;
  if (use_smem) {
    for (int t = threadIdx.x; t < nseg * nD; t += blockDim.x) s_part[t] = 0.0;
    __syncthreads();
  }
  const int nch = (nvalid + CH - 1) / CH;
  for (int it = threadIdx.x; it < nch * nD; it += blockDim.x) {
    const int d = it % nD, c = it / nD;
    const int l0 = c * CH, l1 = min(l0 + CH, nvalid);
    int f = (int)((g0 + l0) / p.Mt);
    int bnd = (int)((long)(f + 1) * p.Mt - g0);  // local index of the next frame's first window
    double s = 0.0;
    for (int l = l0; l < l1; l++) {
      if (l == bnd) {
        if (s > 0.0) {
          if (use_smem) atomicAdd(s_part + (f - f0) * nD + d, s);
          else atomicAdd(p.Lacc + ((size_t)f * p.N + i) * p.q + D0 + d, s);
        }
        s = 0.0;
        f++;
        bnd += p.Mt;
      }
      const double w = s_w[l];
      if (w > 0.0) s += w * (double)s_t[l * ts + d];
    }
    if (s > 0.0) {
      if (use_smem) atomicAdd(s_part + (f - f0) * nD + d, s);
      else atomicAdd(p.Lacc + ((size_t)f * p.N + i) * p.q + D0 + d, s);
    }
  }
  if (use_smem) {
    __syncthreads();
    for (int t = threadIdx.x; t < nseg * nD; t += blockDim.x) {
      const double v = s_part[t];
      if (v > 0.0) atomicAdd(p.Lacc + ((size_t)(f0 + t / nD) * p.N + i) * p.q + D0 + t % nD, v);
    }
  }
}

// Per-lane weights of the APP pass: beta_{i+1}(m'+k) rescaled by its max over
// the corridor (FP32 copy in [0,1]) and w = alpha_i(m') * that max (FP64).
template <int MN>
__device__ __forceinline__ double app_weights(const DecodeParams& p, const LaneGeom& G, int i, float (&bt)[MN]) {
  double bm = 0.0;
  double bv[MN];
  const double* brow = beta_row(p, G.f, i + 1);
#pragma unroll
  for (int e = 0; e < MN; e++) {
    bv[e] = out_valid(p, G, e) ? brow[G.mi + p.mn_lo + e] : 0.0;
    bm = fmax(bm, bv[e]);
  }
  const double inv = bm > 0.0 ? 1.0 / bm : 0.0;
#pragma unroll
  for (int e = 0; e < MN; e++) bt[e] = (float)(bv[e] * inv);
  return G.active ? p.alpha[((size_t)G.f * (p.N + 1) + i) * p.Mt + G.mi] * bm : 0.0;
}

// smem: s_w[blockDim] (double) | s_part[kAppSegCap][min(q, kAppDChunk)] (double)
//       | s_t[blockDim][ts] (float) | s_C[q]
template <class Core>
__global__ void __launch_bounds__(kLatticeThreads, kLatticeMinBlocks) k_app(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  extern __shared__ __align__(128) unsigned char smem[];
  const int ts = app_tstride(p.q);
  double* s_w = reinterpret_cast<double*>(smem);
  double* s_part = s_w + blockDim.x;
  float* s_t = reinterpret_cast<float*>(s_part + kAppSegCap * min(p.q, kAppDChunk));
  uint32_t* s_C = reinterpret_cast<uint32_t*>(s_t + (size_t)ts * blockDim.x);
  const int i = blockIdx.y + p.i_base;
  for (int t = threadIdx.x; t < p.q; t += blockDim.x) s_C[t] = p.C[(size_t)i * p.q + t];

  const LaneGeom G = lane_geom(p, i);
  float bt[MN];
  const double w = app_weights<MN>(p, G, i, bt);
  s_w[threadIdx.x] = w;
  __syncthreads();
  const bool warp_live = __any_sync(0xffffffffu, w > 0.0);
  typename Core::Lane lane;
  Core::init(lane, G.active ? load_window(p, G.f, G.s, G.rho) : 0ull, p);
  const float* pri = p.priors ? p.priors + ((size_t)G.f * p.N + i) * p.q : nullptr;

  for (int D0 = 0; D0 < p.q; D0 += kAppDChunk) {
    const int nD = min(kAppDChunk, p.q - D0);
    if (warp_live) {
      for (int d = 0; d < nD; d++) {
        const float P = pri ? __ldg(pri + D0 + d) : 1.f;
        float fo[MN];
        Core::run(lane, s_C[D0 + d], p, fo);
        // t(m', D) = sum_k gamma_i(m', m'+k, D) beta_{i+1}(m'+k) / bmax  (two chains for ILP)
        float t0 = 0.f, t1 = 0.f;
#pragma unroll
        for (int e = 0; e < MN; e += 2) {
          t0 = fmaf(fo[e], bt[e], t0);
          if (e + 1 < MN) t1 = fmaf(fo[e + 1], bt[e + 1], t1);
        }
        s_t[threadIdx.x * ts + d] = P * (t0 + t1);
      }
    }
    __syncthreads();
    app_reduce(p, i, D0, nD, s_w, s_t, ts, (long)blockIdx.x * blockDim.x, blockDim.x, s_part);
    __syncthreads();
  }
}

// Stored variant APP: gamma streamed from HBM instead of recomputed.
// smem: s_w[blockDim] | s_part[kAppSegCap][min(q, kAppDChunk)] | s_t[blockDim][ts]
template <int MN>
__global__ void __launch_bounds__(kLatticeThreads) k_app_stored(const DecodeParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int ts = app_tstride(p.q);
  double* s_w = reinterpret_cast<double*>(smem);
  double* s_part = s_w + blockDim.x;
  float* s_t = reinterpret_cast<float*>(s_part + kAppSegCap * min(p.q, kAppDChunk));
  const int i = blockIdx.y + p.i_base;
  const LaneGeom G = lane_geom(p, i);
  float bt[MN];
  const double w = app_weights<MN>(p, G, i, bt);
  s_w[threadIdx.x] = w;
  const float* gin = p.gamma + (((size_t)G.f * p.N + i) * p.q) * MN * p.Mt + G.mi;
  for (int D0 = 0; D0 < p.q; D0 += kAppDChunk) {
    const int nD = min(kAppDChunk, p.q - D0);
    if (w > 0.0) {
      for (int d = 0; d < nD; d++) {
        const float* gd = gin + (size_t)(D0 + d) * MN * p.Mt;
        float t0 = 0.f, t1 = 0.f;
#pragma unroll
        for (int e = 0; e < MN; e += 2) {
          t0 = fmaf(__ldcs(gd + (size_t)e * p.Mt), bt[e], t0);
          if (e + 1 < MN) t1 = fmaf(__ldcs(gd + (size_t)(e + 1) * p.Mt), bt[e + 1], t1);
        }
        s_t[threadIdx.x * ts + d] = t0 + t1;  // gamma already carries the prior
      }
    }
    __syncthreads();
    app_reduce(p, i, D0, nD, s_w, s_t, ts, (long)blockIdx.x * blockDim.x, blockDim.x, s_part);
    __syncthreads();
  }
}

template <class Core>
__global__ void __launch_bounds__(kLatticeThreads) k_gamma_dump(const DecodeParams p) {
  constexpr int MN = Core::Mn;
  extern __shared__ uint32_t s_C[];
  const int i = p.dbg_i;
  for (int t = threadIdx.x; t < p.q; t += blockDim.x) s_C[t] = p.C[(size_t)i * p.q + t];
  __syncthreads();
  const LaneGeom G = lane_geom(p, i);
  if (!G.in) return;
  typename Core::Lane lane;
  Core::init(lane, G.active ? load_window(p, G.f, G.s, G.rho) : 0ull, p);
  const double unscale = p.lc.out_scale;
  double* out = p.dbg_gamma + ((size_t)G.f * p.Mt + G.mi) * MN * p.q;
  for (int D = 0; D < p.q; D++) {
    const double P = p.priors ? (double)p.priors[((size_t)G.f * p.N + i) * p.q + D] : 1.0 / p.q;
    float fo[MN];
    Core::run(lane, s_C[D], p, fo);
#pragma unroll
    for (int e = 0; e < MN; e++) out[(size_t)e * p.q + D] = out_valid(p, G, e) ? P * (double)fo[e] * unscale : 0.0;
  }
}

// Kernel table for one lattice core.
struct CoreKernels {
  void (*gamma_sum)(const DecodeParams);
  void (*gamma_sum_k3)(const DecodeParams);  // pass 1 with 3 hoisted rows (large q); nullptr = none
  void (*gamma_sum_pri)(const DecodeParams);     // the same two with non-uniform priors (nullptr: the
  void (*gamma_sum_k3_pri)(const DecodeParams);  // plain kernels read priors themselves)
  void (*gamma_store)(const DecodeParams);
  void (*app)(const DecodeParams);
  int app_ks_auto;                         // default folded rows of this core's APP kernel
  void (*app_live[2][4])(const DecodeParams);  // live-window APP [KS - 1][KP = 0, 2, 3, 4] (spec only)
  int app_live_W;                          // its windows per lane (1 scalar, 2 pair core)
  size_t l1_head_bytes[2];                 // pass-1 head-table smem of the K = 2, 3 class kernels
  void (*app_stored)(const DecodeParams);
  void (*gamma_dump)(const DecodeParams);
  long nodes;  // corridor nodes per lattice (0 = generic core: computed on host)
  int W;       // windows per lane (1 scalar core, 2 packed-pair core)
  int l1_W;    // windows per lane of the pass-1 kernel (the scalar core may serve pass 1 of a pair core)
  bool l1_steps;  // the pass-1 (non-stored) kernels walk kL1Steps symbol indices per CTA
  void (*ab_warp[3])(const DecodeParams);  // warp-per-task alpha/beta for M_tau <= 32, 64, 128 (spec only)
  void (*ab_cta)(const DecodeParams, int);  // CTA-per-task alpha/beta with compile-time M_n (spec only)
  void (*local_fwd)(const DecodeParams);   // fused local schedule, M_tau <= 64 (spec only)
  void (*local_cta_fwd[2][2])(const DecodeParams);  // CTA-per-frame local schedule [K - 2][priors] (spec only)
  void (*local_cta_bwd[2])(const DecodeParams);     // [priors]
  void (*local_bwd)(const DecodeParams);
};

template <class Core>
CoreKernels make_core_kernels(long nodes) {
  CoreKernels k{};
  k.gamma_sum = k_gamma_sum<Core, false>;
  k.gamma_sum_k3 = nullptr;
  k.gamma_sum_pri = k.gamma_sum_k3_pri = nullptr;
  k.gamma_store = k_gamma_sum<Core, true>;
  k.app = k_app<Core>;
  k.app_ks_auto = 1;
  for (auto& r : k.app_live)
    for (auto& fn : r) fn = nullptr;
  k.app_live_W = 0;
  k.l1_head_bytes[0] = k.l1_head_bytes[1] = 0;
  k.app_stored = k_app_stored<Core::Mn>;
  k.gamma_dump = k_gamma_dump<Core>;
  k.nodes = nodes;
  k.W = 1;
  k.l1_W = 1;
  k.ab_warp[0] = k.ab_warp[1] = k.ab_warp[2] = nullptr;
  k.local_fwd = k.local_bwd = nullptr;
  k.ab_cta = nullptr;
  k.l1_steps = false;
  k.local_cta_fwd[0][0] = k.local_cta_fwd[0][1] = k.local_cta_fwd[1][0] = k.local_cta_fwd[1][1] = nullptr;
  k.local_cta_bwd[0] = k.local_cta_bwd[1] = nullptr;
  return k;
}

#ifndef __CUDACC_RTC__
// Registry (defined in the instantiation units) and the run-time compiled shapes (jit.cu).
bool find_spec_kernels(int n, int mn_lo, int Mn, CoreKernels* out);
bool find_generic_kernels(int Mn, CoreKernels* out);
bool jit_spec_kernels(int n, int mn_lo, int Mn, CoreKernels* out, std::string* err, bool compile_only);
#endif

}  // namespace bsidmap
