// Expansion-kernel instruction mix vs the FP64 pipe, full GPU (2048 CTAs x 256 threads,
// 2 CTAs/SM): MODE 0 pure DFMA (32 independent chains per thread), MODE 1 + one LDS.128
// broadcast per 4 DFMA, MODE 2 + the +-1.0 kappa construction (SHL, LOP3, MOV per column-term).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(256, 2) k(double* out, int iters, unsigned seed) {
  __shared__ __align__(16) double rho[16][32];
  for (int i = threadIdx.x; i < 16 * 32; i += 256) rho[i / 32][i % 32] = 1e-3 * (i + 1);
  __syncthreads();
  double acc[16][2];
  for (int r = 0; r < 16; ++r) acc[r][0] = acc[r][1] = threadIdx.x;
  unsigned v0 = seed ^ threadIdx.x, v1 = seed * 7 + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 0; b < 32; b += 2) {
      double k00 = 1.0, k01 = -1.0, k10 = 1.0, k11 = -1.0;
      if (MODE == 2) {
        k00 = __hiloint2double((int)(0x3FF00000u | ((v0 << (31 - b)) & 0x80000000u)), 0);
        k01 = __hiloint2double((int)(0x3FF00000u | ((v0 << (30 - b)) & 0x80000000u)), 0);
        k10 = __hiloint2double((int)(0x3FF00000u | ((v1 << (31 - b)) & 0x80000000u)), 0);
        k11 = __hiloint2double((int)(0x3FF00000u | ((v1 << (30 - b)) & 0x80000000u)), 0);
      }
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        double2 x;
        if (MODE == 0) { x.x = 1e-9 * (r + b); x.y = -1e-9 * (r + b); }
        else {  // volatile shared load: the compiler may not hoist it out of the iteration loop
          const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&rho[r][b]));
          asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x.x), "=d"(x.y) : "r"(sa));
        }
        acc[r][0] = fma(k00, x.x, acc[r][0]);
        acc[r][1] = fma(k10, x.x, acc[r][1]);
        acc[r][0] = fma(k01, x.y, acc[r][0]);
        acc[r][1] = fma(k11, x.y, acc[r][1]);
      }
    }
    v0 = v0 * 1664525u + 1013904223u;
    v1 = v1 * 22695477u + 1u;
  }
  double s = 0;
  for (int r = 0; r < 16; ++r) s += acc[r][0] + acc[r][1];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}
template <int MODE>
void run(const char* name) {
  double* out; cudaMalloc(&out, 2048 * 256 * 8);
  int iters = 512;
  k<MODE><<<2048, 256>>>(out, 8, 1);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<2048, 256>>>(out, iters, 1);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double dfma = 2048.0 * 256 * iters * 32 * 32;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double peak = 64.0 * 148 * 1.965e9;
  printf("%-28s %.3f ms  %.2f TDFMA/s  frac of 64/clk/SM @1965 MHz: %.3f\n", name, ms, dfma / (ms * 1e-3) / 1e12,
         dfma / (ms * 1e-3) / peak);
  cudaFree(out);
}
int main() {
  run<0>("pure DFMA");
  run<1>("DFMA + LDS.128 per 4");
  run<2>("DFMA + LDS + kappa");
  return 0;
}
