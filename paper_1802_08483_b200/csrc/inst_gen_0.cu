// Generic lattice cores (runtime n, m_n^-) for M_n = 1..8.
#include "inst.cuh"
namespace bsidmap {
bool gen_unit_0(int Mn, CoreKernels* out) {
  switch (Mn) {
    BSIDMAP_GEN_CASE(1)
    BSIDMAP_GEN_CASE(2)
    BSIDMAP_GEN_CASE(3)
    BSIDMAP_GEN_CASE(4)
    BSIDMAP_GEN_CASE(5)
    BSIDMAP_GEN_CASE(6)
    BSIDMAP_GEN_CASE(7)
    BSIDMAP_GEN_CASE(8)
  }
  return false;
}
}  // namespace bsidmap
