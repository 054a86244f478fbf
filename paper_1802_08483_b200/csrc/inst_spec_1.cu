// Fully unrolled lattice core for (n, m_n^-, M_n) = (10,-6,13).
#include "inst.cuh"
BSIDMAP_SPEC_UNIT(1, 10,-6,13)
