// RELOAD variant prototype: RG rows per step, rows re-read from SMEM in step B.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ double flipd(double x, unsigned m) { return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x)); }
__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(saddr(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(saddr(b)) : "memory"); }
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned ph) { unsigned ok; asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(saddr(b)), "r"(ph) : "memory"); return ok; }
template <int RG>
__device__ __forceinline__ double wred(double (&p)[RG], int lane) {
  if constexpr (RG == 1) { double v = p[0]; for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(~0u, v, o); return v; }
  else if constexpr (RG == 2) { const bool up = lane & 16; double v = (up ? p[1] : p[0]) + __shfl_xor_sync(~0u, up ? p[0] : p[1], 16);
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(~0u, v, o); return v; }
  else { const bool up = lane & 16;
    const double q0 = (up ? p[2] : p[0]) + __shfl_xor_sync(~0u, up ? p[0] : p[2], 16);
    const double q1 = (up ? p[3] : p[1]) + __shfl_xor_sync(~0u, up ? p[1] : p[3], 16);
    const bool b3 = lane & 8; double v = (b3 ? q1 : q0) + __shfl_xor_sync(~0u, b3 ? q0 : q1, 8);
    for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(~0u, v, o); return v; }
}
template <int RG> __device__ __forceinline__ int hl(int r) { return RG == 1 ? 0 : (RG == 2 ? r * 16 : (r >> 1) * 16 + (r & 1) * 8); }
template <int NW, int VPT, int RG, int MODE>
__global__ void __launch_bounds__((NW + 1) * 32, 1) k(int rows, int passes, long long* cyc, double* out) {
  constexpr int NE = VPT * 4;
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = 4096, NV = n / 4;
  float4* R = reinterpret_cast<float4*>(smem);
  double* rred = reinterpret_cast<double*>(smem + rows * n * 4);
  unsigned long long* ring = reinterpret_cast<unsigned long long*>(rred + 4 * RG * NW);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < rows * NV; i += blockDim.x) R[i] = make_float4(i * 1e-3f, -i * 2e-3f, 0.5f, -0.25f);
  if (tid == 0) for (int s = 0; s < 4; ++s) mbar_init(&ring[s], NW);
  __syncthreads();
  if (warp >= NW) return;
  unsigned tbits = 0x5a5a5a5au ^ tid;
  double zacc[NE];
  for (int i = 0; i < NE; ++i) zacc[i] = 0;
  unsigned gc = 0;
  const int ng = rows / RG;
  long long t0 = clock64();
  auto A = [&](int g) {
    float x[RG][NE];
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const float4* rv = R + (g * RG + r) * NV;
#pragma unroll
      for (int kk = 0; kk < VPT; ++kk) { float4 v = rv[(kk * NW + warp) * 32 + lane]; x[r][kk*4]=v.x; x[r][kk*4+1]=v.y; x[r][kk*4+2]=v.z; x[r][kk*4+3]=v.w; }
    }
    unsigned tb = tbits; asm volatile("" : "+r"(tb));
    double p[RG];
#pragma unroll
    for (int r = 0; r < RG; ++r) { double ac[4] = {0,0,0,0};
#pragma unroll
      for (int i = 0; i < NE; ++i) ac[i & 3] += flipd((double)x[r][i], (tb << (31 - i)) & 0x80000000u); p[r] = (ac[0]+ac[1])+(ac[2]+ac[3]); }
    if (MODE & 2) { if (lane == 0) for (int r = 0; r < RG; ++r) rred[r] = p[r]; return; }
    const double v = wred<RG>(p, lane);
    const unsigned gi = gc + g;
#pragma unroll
    for (int r = 0; r < RG; ++r) if (lane == hl<RG>(r)) rred[((gi & 3) * RG + r) * NW + warp] = v;
    if (MODE & 4) return;
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring[gi & 3]);
  };
  auto B = [&](int g) {
    const unsigned gi = gc + g;
    while (!mbar_try(&ring[gi & 3], (gi >> 2) & 1)) {}
    double y = 0;
    if (lane < RG) {
      const double* pr = rred + ((gi & 3) * RG + lane) * NW;
      double y0 = 0, y1 = 0;
#pragma unroll
      for (int w = 0; w < NW; w += 2) { y0 += pr[w]; y1 += pr[w + 1]; }
      y = y0 + y1;
    }
    const unsigned nb = __ballot_sync(~0u, lane < RG && y < 0);
#pragma unroll
    for (int r = 0; r < RG; ++r) {
      const float4* rv = R + (g * RG + r) * NV;
      float x[NE];
#pragma unroll
      for (int kk = 0; kk < VPT; ++kk) { float4 v = rv[(kk * NW + warp) * 32 + lane]; x[kk*4]=v.x; x[kk*4+1]=v.y; x[kk*4+2]=v.z; x[kk*4+3]=v.w; }
      if ((nb >> r) & 1) {
#pragma unroll
        for (int i = 0; i < NE; ++i) zacc[i] -= (double)x[i];
      } else {
#pragma unroll
        for (int i = 0; i < NE; ++i) zacc[i] += (double)x[i];
      }
    }
  };
  for (int P = 0; P < passes; ++P) {
    A(0);
    for (int g = 1; g < ng; ++g) { A(g); if (!(MODE & 1)) B(g - 1); }
    if (!(MODE & 1)) B(ng - 1);
    gc += ng;
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0; for (int i = 0; i < NE; ++i) s += zacc[i];
  out[blockIdx.x * 288 + tid] = s;
}
template <int NW, int VPT, int RG, int MODE> void run(const char* nm) {
  int rows = 12, passes = 200; size_t sm = rows * 4096 * 4 + 4 * RG * NW * 8 + 64;
  auto f = k<NW, VPT, RG, MODE>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  long long* cyc; double* out; cudaMalloc(&cyc, 8 * 148); cudaMalloc(&out, 8 * 148 * 1024);
  f<<<148, (NW + 1) * 32, sm>>>(rows, passes, cyc, out); cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148); cudaMemcpy(h.data(), cyc, 8 * 148, cudaMemcpyDeviceToHost);
  double a = 0; for (auto v : h) a += v; a /= 148.0 * passes * rows;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, f);
  printf("%-24s %7.0f cycles/row  regs=%d local=%zu (%s)\n", nm, a, fa.numRegs, fa.localSizeBytes, cudaGetErrorString(e));
}
int main() {
  run<8, 4, 4, 3>("RG4 A: no tree/publish");
  run<8, 4, 4, 5>("RG4 A: tree+STS, no arrive");
  run<8, 4, 4, 1>("RG4 A: tree+STS+arrive");
  run<8, 4, 1, 3>("RG1 A: no tree/publish");
  run<8, 4, 1, 5>("RG1 A: tree+STS, no arrive");
  run<8, 4, 1, 1>("RG1 A: tree+STS+arrive");
  return 0;
}
