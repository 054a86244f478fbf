// inst.cuh -- explicit instantiation helpers (split over compilation units so
// nvcc compiles the unrolled lattice cores in parallel).
#pragma once
#include "k_local_x2.cuh"

#define BSIDMAP_SPEC_UNIT(IDX, NN, LO, MN)                                               \
  namespace bsidmap {                                                                    \
  bool spec_unit_##IDX(int n, int lo, int Mn, CoreKernels* out) {                        \
    if (n != NN || lo != LO || Mn != MN) return false;                                   \
    *out = make_core_kernels_x2<SpecCoreX2<NN, LO, MN>>(SpecCoreX2<NN, LO, MN>::nodes()); \
    return true;                                                                         \
  }                                                                                      \
  }

#define BSIDMAP_GEN_CASE(MN) \
  case MN: *out = make_core_kernels<GenCore<MN>>(0); return true;
