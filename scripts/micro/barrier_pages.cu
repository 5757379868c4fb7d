// Is the flat grid barrier's cost a function of the 2 MB page its counter lives
// in (and of the L2 state a preceding 256 MB write leaves)?  One counter per
// candidate page of a 128 MB allocation; 148 CTAs x 2000 barriers on each.
// Also times a "slots" pattern: every CTA stores one line and, after the
// barrier, reads all 148 lines (the sweep kernel's pass-end exchange).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <bool SLOTS>
__global__ void k(unsigned* ctr, double* slots, int rounds, double* sink) {
  const int g = blockIdx.x, G = gridDim.x;
  unsigned ep = 0;
  double acc = 0.0;
  for (int P = 0; P < rounds; ++P) {
    if (SLOTS && threadIdx.x == 0) __stcg(slots + g * 16 + (P & 1), static_cast<double>(P + g));
    __syncthreads();
    if (threadIdx.x == 0) {
      ++ep;
      red_rel(ctr, 1);
      while (static_cast<int>(ld_rlx(ctr) - ep * G) < 0) {
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
    if (SLOTS)
      for (int i = threadIdx.x; i < G; i += blockDim.x) acc += __ldcg(slots + i * 16 + (P & 1));
  }
  if (acc == -1.0) sink[g] = acc;
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t span = 128ull << 20, page = 2ull << 20;
  char* mem;
  char* flush;
  double* sink;
  cudaMalloc(&mem, span);
  cudaMalloc(&flush, 256ull << 20);
  cudaMalloc(&sink, 8 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int rounds = 2000;
  for (int fl = 0; fl < 2; ++fl) {
    for (int slots = 0; slots < 2; ++slots) {
      printf("flush=%d slots=%d us/barrier per page:", fl, slots);
      for (size_t off = 0; off < span; off += page) {
        unsigned* ctr = reinterpret_cast<unsigned*>(mem + off);
        double* sl = reinterpret_cast<double*>(mem + off + 4096);
        float best = 1e9f;
        for (int rep = 0; rep < 2; ++rep) {
          cudaMemset(ctr, 0, 256);
          if (fl) cudaMemset(flush, rep, 256ull << 20);
          void* args[] = {&ctr, &sl, &rounds, &sink};
          cudaEventRecord(a);
          cudaLaunchCooperativeKernel(slots ? (void*)k<true> : (void*)k<false>, sms, 256, args, 0, 0);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        printf(" %.2f", best * 1e3 / rounds);
      }
      printf("\n");
      fflush(stdout);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
