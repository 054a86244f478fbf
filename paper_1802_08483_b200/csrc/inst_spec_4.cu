// Fully unrolled lattice core for (n, m_n^-, M_n) = (12,-7,16).
#include "inst.cuh"
BSIDMAP_SPEC_UNIT(4, 12,-7,16)
