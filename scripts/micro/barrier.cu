// Grid barrier latency: 148 CTAs, atomics + acquire spin, with/without fences.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(unsigned* bar, int rounds, long long* cyc) {
  unsigned epoch = 0;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      ++epoch;
      const unsigned target = epoch * gridDim.x;
      if (MODE == 0) { __threadfence(); atomicAdd(bar, 1u); while ((int)(*(volatile unsigned*)bar - target) < 0) {} __threadfence(); }
      if (MODE == 1) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(bar) : "memory");
        unsigned v; do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while ((int)(v - target) < 0);
      }
      if (MODE == 2) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(bar) : "memory");
        unsigned v; do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while ((int)(v - target) < 0);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}
int main() {
  unsigned* bar; long long* cyc; cudaMalloc(&bar, 4); cudaMalloc(&cyc, 8 * 1024);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int rounds = 10000;
  for (int mode = 0; mode < 3; ++mode) for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(bar, 0, 4);
    void* args[] = {&bar, &rounds, &cyc};
    cudaEventRecord(a);
    if (mode == 0) cudaLaunchCooperativeKernel((void*)k<0>, sms, 256, args, 0, 0);
    if (mode == 1) cudaLaunchCooperativeKernel((void*)k<1>, sms, 256, args, 0, 0);
    if (mode == 2) cudaLaunchCooperativeKernel((void*)k<2>, sms, 256, args, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("mode %d: %.3f us per grid barrier (err=%s)\n", mode, ms * 1e3 / rounds, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
