// Per-row dot+z work with rows in SMEM: compares f32->f64 widening strategies.
// CONV 0: F2F for the dot and again for z (current kernel)
// CONV 1: F2F once, f64 kept in registers for z
// CONV 2: integer widening (ALU/IMAD, exact for normals and zero), kept for z
// CONV 3: integer widening for the dot, F2F for z (splits MIO vs ALU)
// RED  0: 5-level shfl.f64 butterfly per row; 1: no cross-lane reduction
#include <cstdio>
#include <vector>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ double flipd(double x, unsigned m) { return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x)); }
__device__ __forceinline__ double widen_alu(uint32_t u) {
  const uint32_t a = u & 0x7fffffffu;
  uint32_t h = __umulhi(a, 1u << 29) + 0x38000000u;
  h = a ? h : 0u;
  return __hiloint2double(static_cast<int>(h | (u & 0x80000000u)), static_cast<int>(u << 29));
}
template <int NW, int VPT, int CONV, int RED>
__global__ void __launch_bounds__(NW * 32, 1) k(int rows, int passes, long long* cyc, double* out) {
  constexpr int NE = VPT * 4;
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = 4096, NV = n / 4;
  float4* R = reinterpret_cast<float4*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < rows * NV; i += blockDim.x) R[i] = make_float4(i * 1e-3f, -i * 2e-3f, 0.5f, -0.25f);
  __syncthreads();
  const unsigned tbits = 0x5a5a5a5au ^ (tid * 2654435761u);
  uint32_t fm[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) fm[i] = (tbits << (31 - i)) & 0x80000000u;
  double zacc[NE];
#pragma unroll
  for (int i = 0; i < NE; ++i) zacc[i] = 0;
  double ysum = 0;
  long long t0 = clock64();
  for (int P = 0; P < passes; ++P) {
    for (int j = 0; j < rows; ++j) {
      const float4* rv = R + j * (size_t)NV;
      float x[NE];
#pragma unroll
      for (int kk = 0; kk < VPT; ++kk) {
        float4 v = rv[(kk * NW + warp) * 32 + lane];
        x[kk * 4] = v.x; x[kk * 4 + 1] = v.y; x[kk * 4 + 2] = v.z; x[kk * 4 + 3] = v.w;
      }
      double xd[NE];
      double ac[4] = {0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < NE; ++i) {
        if (CONV == 0 || CONV == 1) {
          xd[i] = (double)x[i];
          ac[i & 3] += flipd(xd[i], fm[i]);
        } else {
          const uint32_t u = __float_as_uint(x[i]);
          xd[i] = widen_alu(u);
          ac[i & 3] += widen_alu(u ^ fm[i]);
        }
      }
      double v = (ac[0] + ac[1]) + (ac[2] + ac[3]);
      if (RED == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      }
      ysum += v;
      const bool neg = __shfl_sync(0xffffffffu, v, 0) < 0.0;
      if (neg) {
#pragma unroll
        for (int i = 0; i < NE; ++i) zacc[i] -= (CONV == 0 || CONV == 3) ? (double)x[i] : xd[i];
      } else {
#pragma unroll
        for (int i = 0; i < NE; ++i) zacc[i] += (CONV == 0 || CONV == 3) ? (double)x[i] : xd[i];
      }
    }
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  double s = ysum;
#pragma unroll
  for (int i = 0; i < NE; ++i) s += zacc[i];
  out[blockIdx.x * 1024 + tid] = s;
}
template <int NW, int VPT, int CONV, int RED> void run(const char* nm) {
  int rows = 12, passes = 100; size_t sm = rows * 4096 * 4;
  auto f = k<NW, VPT, CONV, RED>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  long long* cyc; double* out; cudaMalloc(&cyc, 8 * 148); cudaMalloc(&out, 8 * 148 * 1024);
  f<<<148, NW * 32, sm>>>(rows, passes, cyc, out); cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148); cudaMemcpy(h.data(), cyc, 8 * 148, cudaMemcpyDeviceToHost);
  double a = 0; for (auto v : h) a += v; a /= 148.0 * passes * rows;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, f);
  printf("NW=%d VPT=%d %-34s %6.0f cycles/row %5.1f elem/clk/SM regs=%d lmem=%zu (%s)\n", NW, VPT, nm, a, 4096 / a,
         fa.numRegs, fa.localSizeBytes, cudaGetErrorString(e));
  cudaFree(cyc); cudaFree(out);
}
#define R4(NW, VPT)                                   \
  run<NW, VPT, 0, 0>("F2F x2 (current) +shfl");        \
  run<NW, VPT, 1, 0>("F2F once kept +shfl");           \
  run<NW, VPT, 2, 0>("ALU widen kept +shfl");          \
  run<NW, VPT, 3, 0>("ALU dot, F2F z +shfl");          \
  run<NW, VPT, 0, 1>("F2F x2 (current) no-red");       \
  run<NW, VPT, 1, 1>("F2F once kept no-red");          \
  run<NW, VPT, 2, 1>("ALU widen kept no-red");
int main() {
  R4(8, 4)
  R4(4, 8)
  R4(16, 2)
  return 0;
}
