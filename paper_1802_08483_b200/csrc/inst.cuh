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

// pass 1 of those shapes stays on the pair class kernel at 3 CTAs/SM (k_lattice_x2.cuh; the scalar
// class kernel measured slower: tools/exp_p1x2.sh)

#define BSIDMAP_SPEC_UNIT(IDX, NN, LO, MN)                                               \
  namespace bsidmap {                                                                    \
  bool spec_unit_##IDX(int n, int lo, int Mn, CoreKernels* out) {                        \
    if (n != NN || lo != LO || Mn != MN) return false;                                   \
    *out = make_core_kernels_x2<SpecCoreX2<NN, LO, MN>>(SpecCoreX2<NN, LO, MN>::nodes()); \
    out->ab_cta = k_alpha_beta_cta<MN>;                                                   \
    local_cta_kernels<SpecCore<NN, LO, MN>>(out);                                          \
    if (SpecCoreX2<NN, LO, MN>::kMinBlocks <= 2 && MN <= BSIDMAP_SCALAR_MN_MAX) { /* measured: scalar APP wins (C3, C5) */ \
      out->app = k_app_x1<SpecCore<NN, LO, MN>, 0>;                                     \
      out->app_pre[0] = k_app_x1<SpecCore<NN, LO, MN>, 2>;                              \
      out->app_pre[1] = k_app_x1<SpecCore<NN, LO, MN>, 3>;                              \
      out->app_pre[2] = k_app_x1<SpecCore<NN, LO, MN>, 4>;                              \
      out->app_ks2 = k_app_x1<SpecCore<NN, LO, MN>, 0, 2>;                              \
      out->app_pre_ks2[0] = k_app_x1<SpecCore<NN, LO, MN>, 2, 2>;                       \
      out->app_pre_ks2[1] = k_app_x1<SpecCore<NN, LO, MN>, 3, 2>;                       \
      out->app_pre_ks2[2] = k_app_x1<SpecCore<NN, LO, MN>, 4, 2>;                       \
      /* fold two rows where the per-symbol tail is short (C3: 90.4 -> 85.6 ms; C5, n = 12: 110 -> 113) */ \
      out->app_ks_auto = NN <= 10 ? 2 : 1;                                              \
      out->app_W = 1;                                                                   \
    }                                                                                   \
    return true;                                                                         \
  }                                                                                      \
  }

#define BSIDMAP_GEN_CASE(MN) \
  case MN: *out = make_core_kernels<GenCore<MN>>(0); return true;
