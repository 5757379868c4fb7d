// Pipe throughput microbenchmark: F2F.F64.F32, DADD, DFMA, FADD, conversions via int.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(const float* in, double* out, int iters) {
  float f[8]; double d[8];
  for (int i = 0; i < 8; ++i) { f[i] = in[(threadIdx.x + i) & 255]; d[i] = f[i]; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) { d[i] += (double)f[i]; f[i] = __int_as_float(__float_as_int(f[i]) ^ 1); }  // F2F + DADD
      if (OP == 1) { d[i] += d[(i + 1) & 7]; }                                                 // DADD
      if (OP == 2) { d[i] = fma(d[i], 1.0000001, d[(i + 3) & 7]); }                            // DFMA
      if (OP == 3) { f[i] += f[(i + 1) & 7]; }                                                 // FADD
      if (OP == 4) { d[i] += (double)f[i]; d[i] += (double)f[(i+1)&7]; f[i] = __int_as_float(__float_as_int(f[i]) ^ 1);}  // 2 F2F
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += d[i] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* in; double* out; cudaMalloc(&in, 1024); cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaMemset(in, 0, 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"F2F+DADD", "DADD", "DFMA", "FADD", "2xF2F+2xDADD"};
  int iters = 4096;
  for (int op = 0; op < 5; ++op) for (int threads : {256, 512, 1024}) {
    auto launch = [&]() {
      if (op == 0) k<0><<<sms, threads>>>(in, out, iters);
      if (op == 1) k<1><<<sms, threads>>>(in, out, iters);
      if (op == 2) k<2><<<sms, threads>>>(in, out, iters);
      if (op == 3) k<3><<<sms, threads>>>(in, out, iters);
      if (op == 4) k<4><<<sms, threads>>>(in, out, iters);
    };
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = double(sms) * threads * iters * 8;
    printf("%-14s threads/SM=%4d  %.3f ms  %.1f Gop/s  %.2f ops/clk/SM @1.9GHz\n", names[op], threads, ms, ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.9e9);
  }
  return 0;
}
