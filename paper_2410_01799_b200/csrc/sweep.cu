// sweep.cu -- host-side variant selection and launch of the persistent fused
// signed-cut kernel (sweep_impl.cuh).  The kernel families are instantiated in
// separate translation units (sweep_k_{f32,f64}{m,t}.cu) that nvcc compiles in
// parallel; this file only dispatches to them.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "sweep.h"

namespace scb {

void* kernel_f32m(const Variant& v);
void* kernel_f32t(const Variant& v);
void* kernel_f64m(const Variant& v);
void* kernel_f64t(const Variant& v);
void* kernel_vr(const Variant& v);
void* kernel_mr(const Variant& v);

namespace {
void* kernel_for(const Variant& v) {
  if (v.mr) return kernel_mr(v);
  if (v.dtype == 0) return v.tensor ? kernel_f32t(v) : kernel_f32m(v);
  return v.tensor ? (v.cps == 1 ? kernel_f64t(v) : nullptr) : kernel_f64m(v);
}
}  // namespace

int pick_variant(int dtype, long long pitch, Variant* v, long long override_code) {
  // nw consumer warps (+1 producer warp); a thread owns vpt 16-byte vectors of
  // every row and keeps two groups of rg rows in registers (current + lagged).
  const int epv = dtype == 0 ? 4 : 2;
  const long long nv = pitch / epv;
  v->dtype = dtype;
  v->cps = 1;
  v->tensor = 0;
  v->mr = 0;
  v->nw = 8;
  if (nv <= 256) {
    v->vpt = 1; v->rg = 4;
  } else if (nv <= 512) {
    v->vpt = 2; v->rg = 2;
  } else if (nv <= 1024) {
    v->vpt = 4; v->rg = dtype == 0 ? 1 : 2;
  } else if (dtype == 0 && nv > 2048 && nv <= 2560) {
    // rows of 8193..10240 f32 (C3's 3000 x 3 trailing block: 9000): whole rows with
    // 16 consumer warps x 5 vectors instead of two column chunks
    v->nw = 16; v->vpt = 5; v->rg = 1;
  } else if (dtype == 0 && nv > 2560 && nv <= 3584) {
    // rows of 10241..14336 f32 (C4's 4096 x 14336 down projection): 16 warps x 7 vectors
    v->nw = 16; v->vpt = 7; v->rg = 1;
  } else if (dtype == 1 && nv > 2048 && nv <= 3584) {
    // rows of 4097..7168 f64: the same 16-warp x 7-vector tile
    v->nw = 16; v->vpt = 7; v->rg = 1;
  } else {
    // nv <= 2048: whole rows; wider: the same tile over column chunks of 2048
    // vectors (8192 f32 / 4096 f64 columns, one TMA stage each, two-phase pass)
    v->vpt = 8; v->rg = 1;
  }
  if (override_code > 0) {  // tuning override nw*1000000 + vpt*10000 + rg*100 + cps (engine option "variant")
    Variant t = *v;
    t.nw = static_cast<int>(override_code / 1000000);
    t.vpt = static_cast<int>((override_code / 10000) % 100);
    t.rg = static_cast<int>((override_code / 100) % 100);
    t.cps = std::max(1, static_cast<int>(override_code % 100));
    if (kernel_for(t) != nullptr && static_cast<long long>(t.nw) * 32 * t.vpt >= nv) *v = t;
  }
  return 0;
}

cudaError_t set_smem_limit(const Variant& v, size_t bytes) {
  void* f = kernel_for(v);
  if (!f) return cudaErrorInvalidValue;
  const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e != cudaSuccess) return e;
  // all of the unified L1/shared array as shared memory (the kernel streams R
  // through TMA, not L1), so co-residency is decided by the real 228 KB
  return cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}

int blocks_per_sm(const Variant& v, size_t smem_bytes) {
  void* f = kernel_for(v);
  int nb = 0, dev = 0, optin = 0;
  if (!f || cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
      set_smem_limit(v, static_cast<size_t>(optin)) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, (v.nw + 1) * 32, smem_bytes) != cudaSuccess)
    return 0;
  return nb;
}

cudaError_t launch_sweep(const Variant& v, const KParams& p, size_t smem_bytes, cudaStream_t st) {
  void* f = kernel_for(v);
  if (!f) return cudaErrorInvalidValue;
  KParams copy = p;
  void* args[] = {&copy};
  return cudaLaunchCooperativeKernel(f, dim3(p.G), dim3((v.nw + 1) * 32), args, smem_bytes, st);
}

bool has_vr(const Variant& v) { return kernel_vr(v) != nullptr; }

cudaError_t set_smem_limit_vr(const Variant& v, size_t bytes) {
  void* f = kernel_vr(v);
  if (!f) return cudaErrorInvalidValue;
  const cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
}

cudaError_t launch_sweep_vr(const Variant& v, const KParamsVR& p, int G, size_t smem_bytes, cudaStream_t st) {
  void* f = kernel_vr(v);
  if (!f) return cudaErrorInvalidValue;
  KParamsVR copy = p;
  void* args[] = {&copy};
  return cudaLaunchCooperativeKernel(f, dim3(G * p.world), dim3((v.nw + 1) * 32), args, smem_bytes, st);
}

}  // namespace scb
