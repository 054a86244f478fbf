// Fully unrolled lattice core for (n, m_n^-, M_n) = (7,-5,12).
#include "inst.cuh"
BSIDMAP_SPEC_UNIT(0, 7,-5,12)
