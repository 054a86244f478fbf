// Generic lattice cores (runtime n, m_n^-) for M_n = 9..16.
#include "inst.cuh"
namespace bsidmap {
bool gen_unit_1(int Mn, CoreKernels* out) {
  switch (Mn) {
    BSIDMAP_GEN_CASE(9)
    BSIDMAP_GEN_CASE(10)
    BSIDMAP_GEN_CASE(11)
    BSIDMAP_GEN_CASE(12)
    BSIDMAP_GEN_CASE(13)
    BSIDMAP_GEN_CASE(14)
    BSIDMAP_GEN_CASE(15)
    BSIDMAP_GEN_CASE(16)
  }
  return false;
}
}  // namespace bsidmap
