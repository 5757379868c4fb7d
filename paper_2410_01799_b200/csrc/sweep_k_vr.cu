// sweep_k_vr.cu -- multi-rank instantiations: the row-sharded rank kernel
// (world > 1, one GPU per rank) and the virtual-rank kernel (row sharding
// emulated on one GPU as one cooperative launch over all ranks' bands;
// sweep.h KParamsVR).  Matrix kernels only, the variants the sharded tests and
// C5 shapes select.
#include "sweep_impl.cuh"

namespace scb {
void* kernel_vr(const Variant& v) {
  if (v.cps != 1 || v.tensor) return nullptr;
#define SCB_K(E, NW, VPT, RG) \
  if (v.nw == NW && v.vpt == VPT && v.rg == RG) return reinterpret_cast<void*>(&sweep_kernel_vr<E, NW, VPT, RG>);
  if (v.dtype == 0) {
    SCB_K(float, 8, 1, 4)
    SCB_K(float, 8, 2, 2)
    SCB_K(float, 8, 4, 1)
    SCB_K(float, 8, 8, 1)
  } else {
    SCB_K(double, 8, 1, 4)
    SCB_K(double, 8, 2, 2)
    SCB_K(double, 8, 4, 2)
    SCB_K(double, 8, 8, 1)
  }
#undef SCB_K
  return nullptr;
}
void* kernel_mr(const Variant& v) {
  if (v.cps != 1 || v.tensor) return nullptr;
#define SCB_K(E, NW, VPT, RG) \
  if (v.nw == NW && v.vpt == VPT && v.rg == RG) return reinterpret_cast<void*>(&sweep_kernel_mr<E, NW, VPT, RG>);
  if (v.dtype == 0) {
    SCB_K(float, 8, 1, 4)
    SCB_K(float, 8, 2, 2)
    SCB_K(float, 8, 4, 1)
    SCB_K(float, 8, 8, 1)
  } else {
    SCB_K(double, 8, 1, 4)
    SCB_K(double, 8, 2, 2)
    SCB_K(double, 8, 4, 2)
    SCB_K(double, 8, 8, 1)
  }
#undef SCB_K
  return nullptr;
}
}  // namespace scb
