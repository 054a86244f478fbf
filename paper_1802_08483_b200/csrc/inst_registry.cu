// inst_registry.cu -- lookup of the compiled lattice cores.
#include "k_lattice.cuh"

namespace bsidmap {
bool spec_unit_0(int, int, int, CoreKernels*);
bool spec_unit_1(int, int, int, CoreKernels*);
bool spec_unit_2(int, int, int, CoreKernels*);
bool spec_unit_3(int, int, int, CoreKernels*);
bool spec_unit_4(int, int, int, CoreKernels*);
bool gen_unit_0(int, CoreKernels*);
bool gen_unit_1(int, CoreKernels*);
bool gen_unit_2(int, CoreKernels*);
bool gen_unit_3(int, CoreKernels*);

bool find_spec_kernels(int n, int lo, int Mn, CoreKernels* out) {
  return spec_unit_0(n, lo, Mn, out) || spec_unit_1(n, lo, Mn, out) || spec_unit_2(n, lo, Mn, out) ||
         spec_unit_3(n, lo, Mn, out) || spec_unit_4(n, lo, Mn, out);
}

bool find_generic_kernels(int Mn, CoreKernels* out) {
  return gen_unit_0(Mn, out) || gen_unit_1(Mn, out) || gen_unit_2(Mn, out) || gen_unit_3(Mn, out);
}
}  // namespace bsidmap
