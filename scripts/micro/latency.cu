// Dependent-chain latencies on sm_100a (single warp): DADD, DFMA, F2F.F64.F32, SHFL (f64 pair), LDS.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, float* fin, long long* cyc, int n) {
  __shared__ double sm[64];
  double d = out[0]; float f = fin[threadIdx.x];
  if (threadIdx.x < 64) sm[threadIdx.x] = d;
  __syncthreads();
  long long t0, t1;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) d = d + 1.0000001;
  t1 = clock64(); cyc[0] = (t1 - t0);
  // F2F chain: f -> d -> f ...
  t0 = clock64();
  for (int i = 0; i < n; ++i) { d = (double)f; f = (float)(d * 1.0); }
  t1 = clock64(); cyc[1] = (t1 - t0);
  // SHFL chain on double
  t0 = clock64();
  for (int i = 0; i < n; ++i) d += __shfl_xor_sync(0xffffffffu, d, 1);
  t1 = clock64(); cyc[2] = (t1 - t0);
  // LDS chain
  int idx = threadIdx.x & 63;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { d = sm[idx]; idx = ((int)d + idx) & 63; }
  t1 = clock64(); cyc[3] = (t1 - t0);
  // FADD chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) f = f + 1.0001f;
  t1 = clock64(); cyc[4] = (t1 - t0);
  out[threadIdx.x + 1] = d + f;
}
int main() {
  double* out; float* fin; long long* cyc;
  cudaMalloc(&out, 8 * 64); cudaMalloc(&fin, 4 * 64); cudaMalloc(&cyc, 8 * 8);
  cudaMemset(out, 0, 8 * 64); cudaMemset(fin, 0, 4 * 64);
  int n = 4096;
  k<<<1, 32>>>(out, fin, cyc, n); cudaDeviceSynchronize();
  k<<<1, 32>>>(out, fin, cyc, n); cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, cyc, 64, cudaMemcpyDeviceToHost);
  const char* nm[] = {"DADD", "F2F f32->f64->f32 (+DMUL)", "SHFL.f64 + DADD", "LDS.64 chain", "FADD"};
  for (int i = 0; i < 5; ++i) printf("%-28s %.1f cycles/iter\n", nm[i], (double)h[i] / n);
  return 0;
}
