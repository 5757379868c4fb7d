// Inner-loop throughput: 8 warps x RG4 x 16 elem/lane, rows in SMEM.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ double flipd(double x, unsigned m) { return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x)); }
template <int NW, int MODE>  // 0: LDS+F2F+flip+DADD 1: LDS+F2F+DADD 2: regs F2F+DADD 3: LDS+FADD 4: LDS only(xor) 5: LDS f64 rows + DADD
__global__ void __launch_bounds__(NW * 32, 1) k(int rows, int passes, long long* cyc, double* out) {
  constexpr int VPT = 32 / NW * 1, NE = VPT * 4, RG = 4;
  extern __shared__ __align__(128) unsigned char smem[];
  const int n = 4096, NV = n / 4;
  float4* R = reinterpret_cast<float4*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < rows * NV; i += blockDim.x) R[i] = make_float4(i * 1e-3f, -i * 2e-3f, 0.5f, -0.25f);
  __syncthreads();
  unsigned tbits = 0x5a5a5a5au ^ tid;
  double acc[RG][4];
  for (int r = 0; r < RG; ++r) for (int i = 0; i < 4; ++i) acc[r][i] = 0;
  float facc[RG][4];
  for (int r = 0; r < RG; ++r) for (int i = 0; i < 4; ++i) facc[r][i] = 0;
  float reg[NE]; for (int i = 0; i < NE; ++i) reg[i] = tid * 0.001f + i;
  unsigned xo = 0;
  long long t0 = clock64();
  for (int P = 0; P < passes; ++P) {
    for (int g = 0; g < rows / RG; ++g) {
      unsigned tb = tbits; asm volatile("" : "+r"(tb));
#pragma unroll
      for (int r = 0; r < RG; ++r) {
        const float4* rv = R + (g * RG + r) * (size_t)NV;
        float x[NE];
        if (MODE == 2) {
#pragma unroll
          for (int i = 0; i < NE; ++i) { x[i] = reg[i]; }
          asm volatile("" : "+f"(x[0]), "+f"(x[1]), "+f"(x[2]), "+f"(x[3]));
        } else {
#pragma unroll
          for (int kk = 0; kk < VPT; ++kk) { float4 v = rv[(kk * NW + warp) * 32 + lane]; x[kk*4]=v.x; x[kk*4+1]=v.y; x[kk*4+2]=v.z; x[kk*4+3]=v.w; }
        }
#pragma unroll
        for (int i = 0; i < NE; ++i) {
          if (MODE == 0) acc[r][i & 3] += flipd((double)x[i], (tb << (31 - i)) & 0x80000000u);
          if (MODE == 1 || MODE == 2) acc[r][i & 3] += (double)x[i];
          if (MODE == 3) facc[r][i & 3] += x[i];
          if (MODE == 4) xo ^= __float_as_uint(x[i]);
        }
      }
    }
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  double s = xo; for (int r = 0; r < RG; ++r) for (int i = 0; i < 4; ++i) s += acc[r][i] + facc[r][i];
  out[blockIdx.x * 1024 + tid] = s;
}
template <int NW, int MODE> void run(const char* nm) {
  int rows = 12, passes = 200; size_t sm = rows * 4096 * 4;
  auto f = k<NW, MODE>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  long long* cyc; double* out; cudaMalloc(&cyc, 8 * 148); cudaMalloc(&out, 8 * 148 * 1024);
  f<<<148, NW * 32, sm>>>(rows, passes, cyc, out); cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148); cudaMemcpy(h.data(), cyc, 8 * 148, cudaMemcpyDeviceToHost);
  double a = 0; for (auto v : h) a += v; a /= 148.0 * passes * rows;
  printf("NW=%2d %-28s %6.0f cycles/row  %5.1f elem/clk/SM (%s)\n", NW, nm, a, 4096 / a, cudaGetErrorString(e));
}
int main() {
  run<8, 0>("LDS+F2F+flip+DADD");
  run<8, 1>("LDS+F2F+DADD");
  run<8, 2>("regs F2F+DADD");
  run<8, 3>("LDS+FADD");
  run<8, 4>("LDS only");
  run<16, 0>("LDS+F2F+flip+DADD");
  run<16, 1>("LDS+F2F+DADD");
  run<16, 2>("regs F2F+DADD");
  run<16, 4>("LDS only");
  run<32, 1>("LDS+F2F+DADD");
  run<32, 4>("LDS only");
  return 0;
}
