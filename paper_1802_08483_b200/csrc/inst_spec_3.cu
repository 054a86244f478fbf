// Fully unrolled lattice core for (n, m_n^-, M_n) = (10,-10,26).
#include "inst.cuh"
BSIDMAP_SPEC_UNIT(3, 10,-10,26)
