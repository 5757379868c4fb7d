// sweep_k_f32m.cu -- f32 matrix instantiations of the sweep kernel (one TU per
// kernel family so the build compiles them in parallel).
#include "sweep_impl.cuh"

namespace scb {
void* kernel_f32m(const Variant& v) {
#define SCB_K(NW, VPT, RG) \
  if (v.nw == NW && v.vpt == VPT && v.rg == RG && v.cps == 1) return reinterpret_cast<void*>(&sweep_kernel<float, NW, VPT, RG, false>);
#define SCB_K2(NW, VPT, RG) \
  if (v.nw == NW && v.vpt == VPT && v.rg == RG && v.cps == 2) return reinterpret_cast<void*>(&sweep_kernel2<float, NW, VPT, RG>);
  SCB_K(8, 1, 4)
  SCB_K(8, 2, 2)
  SCB_K(8, 4, 2)
  SCB_K(8, 4, 1)
  SCB_K(16, 2, 2)
  SCB_K(16, 2, 1)
  SCB_K(8, 8, 1)
  SCB_K(16, 5, 1)
  SCB_K(16, 7, 1)
  SCB_K2(8, 4, 1)
  SCB_K2(8, 2, 2)
#undef SCB_K
#undef SCB_K2
  return nullptr;
}
}  // namespace scb
