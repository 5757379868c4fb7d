#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float* fin, long long* cyc, int n, double* out) {
  float f = fin[threadIdx.x]; double d = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f));
    asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(d));
  }
  long long t1 = clock64(); cyc[0] = t1 - t0;
  // F2F throughput with 8 independent streams per thread
  float g[8]; double e[8];
  for (int j = 0; j < 8; ++j) { g[j] = f + j; e[j] = 0; }
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { double t; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(g[j])); e[j] += t; }
  }
  t1 = clock64(); cyc[1] = t1 - t0;
  double s = d; for (int j = 0; j < 8; ++j) s += e[j];
  out[threadIdx.x] = s + f;
}
int main() {
  float* fin; long long* cyc; double* out;
  cudaMalloc(&fin, 4 * 1024); cudaMalloc(&cyc, 64); cudaMalloc(&out, 8 * 1024);
  cudaMemset(fin, 0, 4096);
  int n = 2048;
  for (int w : {1, 4, 8, 16}) {
    k<<<1, 32 * w>>>(fin, cyc, n, out); cudaDeviceSynchronize();
    k<<<1, 32 * w>>>(fin, cyc, n, out); cudaDeviceSynchronize();
    long long h[2]; cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    printf("warps=%2d  F2F->F2F roundtrip latency %.1f cyc/iter | 8 indep F2F+DADD per iter: %.1f cyc/iter (%.2f warp-F2F/cyc/SM)\n",
           w, (double)h[0] / n, (double)h[1] / n, 8.0 * w / ((double)h[1] / n));
  }
  return 0;
}
