// Generic lattice cores (runtime n, m_n^-) for M_n = 25..32.
#include "inst.cuh"
namespace bsidmap {
bool gen_unit_3(int Mn, CoreKernels* out) {
  switch (Mn) {
    BSIDMAP_GEN_CASE(25)
    BSIDMAP_GEN_CASE(26)
    BSIDMAP_GEN_CASE(27)
    BSIDMAP_GEN_CASE(28)
    BSIDMAP_GEN_CASE(29)
    BSIDMAP_GEN_CASE(30)
    BSIDMAP_GEN_CASE(31)
    BSIDMAP_GEN_CASE(32)
  }
  return false;
}
}  // namespace bsidmap
