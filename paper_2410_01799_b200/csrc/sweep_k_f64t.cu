// sweep_k_f64t.cu -- f64 order-k (tensor) instantiations of the sweep kernel.
#include "sweep_impl.cuh"

namespace scb {
void* kernel_f64t(const Variant& v) {
#define SCB_K(NW, VPT, RG) \
  if (v.nw == NW && v.vpt == VPT && v.rg == RG && v.cps == 1) return reinterpret_cast<void*>(&sweep_kernel<double, NW, VPT, RG, true>);
  SCB_K(8, 1, 4)
  SCB_K(8, 2, 2)
  SCB_K(8, 4, 2)
  SCB_K(8, 8, 1)
  SCB_K(16, 7, 1)
#undef SCB_K
  return nullptr;
}
}  // namespace scb
