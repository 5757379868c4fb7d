// Ablation of the dot-pass row loop (resident rows, 8 warps x 16 elements/lane/row).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ double flipd(double x, unsigned m) { return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x)); }
__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(saddr(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(saddr(b)) : "memory"); }
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned ph) { unsigned ok; asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(saddr(b)), "r"(ph) : "memory"); return ok; }
template <int MODE>  // bits: 1 no F2F (float accum), 2 no shuffle tree, 4 no step B, 8 no ring wait, 16 no publish
__global__ void __launch_bounds__(288, 1) k(int rows, int passes, long long* cyc, double* out) {
  constexpr int NW = 8, VPT = 4, NE = 16;
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = 4096, NV = n / 4;
  float4* R = reinterpret_cast<float4*>(smem);
  double* rred = reinterpret_cast<double*>(smem + rows * n * 4);
  unsigned long long* ring = reinterpret_cast<unsigned long long*>(rred + 4 * NW);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < rows * NV; i += blockDim.x) R[i] = make_float4(i * 1e-3f, -i * 2e-3f, 0.5f, -0.25f);
  if (tid == 0) for (int s = 0; s < 4; ++s) mbar_init(&ring[s], NW);
  __syncthreads();
  if (warp >= NW) return;
  unsigned tbits = 0x5a5a5a5au ^ tid;
  double zacc[NE];
  for (int i = 0; i < NE; ++i) zacc[i] = 0;
  unsigned gc = 0;
  long long t0 = clock64();
  float xa[NE], xb[NE];
  auto A = [&](float (&x)[NE], int j) {
    const float4* rv = R + j * NV;
#pragma unroll
    for (int kk = 0; kk < VPT; ++kk) { float4 v = rv[(kk * NW + warp) * 32 + lane]; x[kk*4]=v.x; x[kk*4+1]=v.y; x[kk*4+2]=v.z; x[kk*4+3]=v.w; }
    double p;
    if (MODE & 1) { float ac[4] = {0,0,0,0}; for (int i = 0; i < NE; ++i) ac[i & 3] += (tbits >> i & 1) ? -x[i] : x[i]; p = (ac[0]+ac[1])+(ac[2]+ac[3]); }
    else { double ac[4] = {0,0,0,0};
#pragma unroll
      for (int i = 0; i < NE; ++i) ac[i & 3] += flipd((double)x[i], (tbits << (31 - i)) & 0x80000000u); p = (ac[0]+ac[1])+(ac[2]+ac[3]); }
    if (!(MODE & 2)) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(~0u, p, o);
    }
    const unsigned gi = gc + j;
    if (!(MODE & 16)) {
      if (lane == 0) { rred[(gi & 3) * NW + warp] = p; mbar_arrive(&ring[gi & 3]); }
    } else if (lane == 0) rred[warp] = p;
  };
  auto B = [&](float (&x)[NE], int j) {
    const unsigned gi = gc + j;
    if (!(MODE & 8) && !(MODE & 16)) while (!mbar_try(&ring[gi & 3], (gi >> 2) & 1)) {}
    double y = 0;
    if (lane == 0) for (int w = 0; w < NW; ++w) y += rred[(gi & 3) * NW + w];
    const unsigned nb = __ballot_sync(~0u, lane == 0 && y < 0);
    if (nb & 1) { for (int i = 0; i < NE; ++i) zacc[i] -= (double)x[i]; } else { for (int i = 0; i < NE; ++i) zacc[i] += (double)x[i]; }
  };
  for (int P = 0; P < passes; ++P) {
    A(xa, 0);
    int g = 1;
    for (; g + 1 < rows; g += 2) {
      A(xb, g); if (!(MODE & 4)) B(xa, g - 1);
      A(xa, g + 1); if (!(MODE & 4)) B(xb, g);
    }
    if (g < rows) { A(xb, g); if (!(MODE & 4)) { B(xa, g - 1); B(xb, g); } } else if (!(MODE & 4)) B(xa, g - 1);
    gc += rows;
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0; for (int i = 0; i < NE; ++i) s += zacc[i];
  out[blockIdx.x * 288 + tid] = s;
}
template <int MODE> void run(const char* nm) {
  int rows = 12, passes = 200; size_t sm = rows * 4096 * 4 + 4 * 8 * 8 + 64;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  long long* cyc; double* out; cudaMalloc(&cyc, 8 * 148); cudaMalloc(&out, 8 * 148 * 288);
  k<MODE><<<148, 288, sm>>>(rows, passes, cyc, out); cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148); cudaMemcpy(h.data(), cyc, 8 * 148, cudaMemcpyDeviceToHost);
  double a = 0; for (auto v : h) a += v; a /= 148.0 * passes * rows;
  printf("%-40s %7.0f cycles/row (%s)\n", nm, a, cudaGetErrorString(e));
}
int main() {
  run<0>("full");
  run<8>("no ring wait");
  run<16>("no publish/wait");
  run<2>("no shuffle tree");
  run<1>("no F2F (float accum in A)");
  run<4>("no step B");
  run<4 | 2>("A only, no tree");
  run<4 | 2 | 1 | 16>("A: loads+float only");
  return 0;
}
