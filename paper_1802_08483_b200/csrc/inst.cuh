// inst.cuh -- explicit instantiation helpers (split over compilation units so
// nvcc compiles the unrolled lattice cores in parallel).
#pragma once
#include "k_local_x2.cuh"
#include "k_alphabeta_cta.cuh"
#include "k_local_cta.cuh"

// register-heavy shapes (pair core at 2 CTAs/SM) with M_n up to this use the scalar core
#ifndef BSIDMAP_SCALAR_MN_MAX
#define BSIDMAP_SCALAR_MN_MAX 20
#endif
// the APP of those shapes on the scalar core (one window per lane)
#ifndef BSIDMAP_SCALAR_APP_MN_MAX
#define BSIDMAP_SCALAR_APP_MN_MAX BSIDMAP_SCALAR_MN_MAX
#endif

// pass 1 of those shapes stays on the pair class kernel at 3 CTAs/SM (k_lattice_x2.cuh; the scalar
// class kernel measured slower: tools/exp_p1x2.sh)

namespace bsidmap {
// Kernel table of one fully unrolled shape (n, m_n^-, M_n).
template <int NN, int LO, int MN>
CoreKernels spec_kernels() {
  CoreKernels k = make_core_kernels_x2<SpecCoreX2<NN, LO, MN>>(SpecCoreX2<NN, LO, MN>::nodes());
  k.ab_cta = k_alpha_beta_cta<MN>;
  local_cta_kernels<SpecCore<NN, LO, MN>>(&k);
  if constexpr (SpecCoreX2<NN, LO, MN>::kMinBlocks <= 2 && MN <= BSIDMAP_SCALAR_APP_MN_MAX) {
    // register-heavy pair shapes: the scalar-core APP measured faster (C3, C5)
    using S = SpecCore<NN, LO, MN>;
    // two folded rows on the scalar core (live-window APP: C3 pass 2 34.5 -> 32.4 ms, C5 26.8 -> 26.4;
    // tools/exp_appkpks.sh)
    k.app_ks_auto = 2;
    k.app_live[0][0] = k_app_live_x1<S, 0, 1>;
    k.app_live[0][1] = k_app_live_x1<S, 2, 1>;
    k.app_live[0][2] = k_app_live_x1<S, 3, 1>;
    k.app_live[0][3] = k_app_live_x1<S, 4, 1>;
    k.app_live[1][0] = k_app_live_x1<S, 0, 2>;
    k.app_live[1][1] = k_app_live_x1<S, 2, 2>;
    k.app_live[1][2] = k_app_live_x1<S, 3, 2>;
    k.app_live[1][3] = k_app_live_x1<S, 4, 2>;
    k.app_live_W = 1;
  }
  return k;
}
}  // namespace bsidmap

#define BSIDMAP_SPEC_UNIT(IDX, NN, LO, MN)                        \
  namespace bsidmap {                                             \
  bool spec_unit_##IDX(int n, int lo, int Mn, CoreKernels* out) { \
    if (n != NN || lo != LO || Mn != MN) return false;            \
    *out = spec_kernels<NN, LO, MN>();                            \
    return true;                                                  \
  }                                                               \
  }

#define BSIDMAP_GEN_CASE(MN) \
  case MN: *out = make_core_kernels<GenCore<MN>>(0); return true;
