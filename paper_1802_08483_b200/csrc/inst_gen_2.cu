// Generic lattice cores (runtime n, m_n^-) for M_n = 17..24.
#include "inst.cuh"
namespace bsidmap {
bool gen_unit_2(int Mn, CoreKernels* out) {
  switch (Mn) {
    BSIDMAP_GEN_CASE(17)
    BSIDMAP_GEN_CASE(18)
    BSIDMAP_GEN_CASE(19)
    BSIDMAP_GEN_CASE(20)
    BSIDMAP_GEN_CASE(21)
    BSIDMAP_GEN_CASE(22)
    BSIDMAP_GEN_CASE(23)
    BSIDMAP_GEN_CASE(24)
  }
  return false;
}
}  // namespace bsidmap
