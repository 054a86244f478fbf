// Fully unrolled lattice core for (n, m_n^-, M_n) = (8,-7,19).
#include "inst.cuh"
BSIDMAP_SPEC_UNIT(2, 8,-7,19)
