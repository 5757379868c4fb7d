// sweep_k_f64m.cu -- f64 matrix instantiations of the sweep kernel.
#include "sweep_impl.cuh"

namespace scb {
void* kernel_f64m(const Variant& v) {
#define SCB_K(NW, VPT, RG) \
  if (v.nw == NW && v.vpt == VPT && v.rg == RG && v.cps == 1) return reinterpret_cast<void*>(&sweep_kernel<double, NW, VPT, RG, false>);
  SCB_K(8, 1, 4)
  SCB_K(8, 2, 2)
  SCB_K(8, 4, 2)
  SCB_K(8, 8, 1)
  SCB_K(16, 4, 1)
  SCB_K(16, 7, 1)
#undef SCB_K
  return nullptr;
}
}  // namespace scb
