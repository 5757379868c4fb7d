// FP64 latency / throughput probes on one SM: dependent DFMA chain, DADD chain,
// independent DFMA streams, IMAD.WIDE+LOP3+DFMA widening stream.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE, int CH>
__global__ void k(double* out, long long* cyc, int iters, double a, int wmul) {
  double acc[CH];
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  unsigned u = threadIdx.x * 2654435761u;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (MODE == 0) acc[c] = fma(acc[c], a, 1.0);
      if (MODE == 1) acc[c] = acc[c] + a;
      if (MODE == 3) {  // F2F + flip + DFMA
        const float f = __uint_as_float((u + c * 977) & 0xbfffffffu);
        const double d = (double)f;
        acc[c] = fma(__hiloint2double(__double2hiint(d) ^ (int)(c << 31), __double2loint(d)), 1.0, acc[c]);
      }
      if (MODE == 4) {  // 32-bit shifts: SHF.R.S32 + LOP3 + SHL
        const unsigned x = u + c * 977;
        const unsigned hi = ((unsigned)((int)x >> 3) & 0x8fffffffu) ^ (c << 31);
        acc[c] = fma(__hiloint2double((int)hi, (int)(x << 29)), 0x1p896, acc[c]);
      }
      if (MODE == 5) {  // compiler-chosen 64-bit shift form (constant multiplier)
        const long long w = (long long)(int)(u + c * 977) * (1ll << 29);
        const unsigned hi = ((unsigned)((unsigned long long)w >> 32) & 0x8fffffffu) ^ (c << 31);
        acc[c] = fma(__hiloint2double((int)hi, (int)(unsigned)w), 0x1p896, acc[c]);
      }
      if (MODE == 2) {
        const long long w = (long long)(int)(u + c * 977) * (long long)wmul;
        const unsigned hi = ((unsigned)((unsigned long long)w >> 32) & 0x8fffffffu) ^ (c << 31);
        acc[c] = fma(__hiloint2double((int)hi, (int)(unsigned)w), 0x1p896, acc[c]);
      }
    }
    u += 7;
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE, int CH> void run(const char* nm, int warps) {
  double* o; long long* c; cudaMalloc(&o, 8 * 148 * 1024); cudaMalloc(&c, 8 * 148);
  int iters = 4096;
  k<MODE, CH><<<148, warps * 32>>>(o, c, iters, 0.999, 1 << 29); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / iters;  // cycles per loop iteration (CH ops per warp)
  printf("%-22s warps=%2d CH=%d: %6.2f cyc/iter  -> %.2f cyc/op/warp, %.1f lanes/clk/SM\n", nm, warps, CH, per, per / CH,
         warps * 32.0 * CH / per);
}
int main() {
  run<0, 1>("DFMA chain", 1);
  run<1, 1>("DADD chain", 1);
  run<0, 8>("DFMA 8 indep", 1);
  run<0, 8>("DFMA 8 indep", 8);
  run<0, 8>("DFMA 8 indep", 16);
  run<1, 8>("DADD 8 indep", 16);
  run<2, 1>("widen+DFMA chain", 1);
  run<2, 8>("widen+DFMA 8", 8);
  run<2, 8>("widen+DFMA 8", 16);
  run<3, 8>("F2F+flip+DFMA 8", 16);
  run<4, 8>("shf32 widen+DFMA 8", 16);
  run<5, 8>("shf64 widen+DFMA 8", 16);
  run<4, 8>("shf32 widen+DFMA 8", 8);
  return 0;
}
