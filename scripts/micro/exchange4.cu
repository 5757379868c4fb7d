// Phase breakdown of the 2-barrier exchange (zpart write, barrier, owner reduce, barrier, read).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void gbar(unsigned* c, unsigned target) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(c) : "memory");
  while ((int)(ld_rlx(c) - target) < 0) {}
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
template <int WRITE, int REDUCE>
__global__ void k(double* zpart, unsigned* tw, unsigned* ctr, int n, int rounds, long long* prof) {
  __shared__ double seg[16][32];
  __shared__ unsigned tws[256];
  const int g = blockIdx.x, G = gridDim.x, tid = threadIdx.x, T = blockDim.x, W = T / 32, lane = tid & 31, warp = tid >> 5;
  const int Q = n / 32;
  unsigned ep = 0; long long t[5] = {0,0,0,0,0}; double acc = 0;
  for (int P = 0; P < rounds; ++P) {
    long long t0 = clock64();
    if (WRITE) for (int c = tid; c < n; c += T) __stcg(zpart + (size_t)g * n + c, (double)((c * 31 + g * 7 + P) % 97) - 48.0);
    __syncthreads();
    long long t1 = clock64();
    if (tid == 0) gbar(ctr, ++ep * G);
    __syncthreads();
    long long t2 = clock64();
    if (REDUCE) for (int q = g; q < Q; q += G) {
      const int gs = warp * G / W, ge = (warp + 1) * G / W;
      double a = 0;
      for (int g0 = gs; g0 < ge; g0 += 16) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = (g0 + u < ge) ? __ldcg(zpart + (size_t)(g0 + u) * n + q * 32 + lane) : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u) a += v[u];
      }
      seg[warp][lane] = a; __syncthreads();
      if (warp == 0) { double z = 0; for (int w = 0; w < W; ++w) z += seg[w][lane]; unsigned b = __ballot_sync(~0u, z < 0); if (lane == 0) __stcg(tw + (P & 1) * 256 + q, b); }
      __syncthreads();
    }
    long long t3 = clock64();
    if (tid == 0) gbar(ctr, ++ep * G);
    __syncthreads();
    long long t4 = clock64();
    for (int i = tid; i < Q; i += T) tws[i] = __ldcg(tw + (P & 1) * 256 + i);
    __syncthreads();
    acc += tws[tid % Q];
    long long t5 = clock64();
    t[0] += t1 - t0; t[1] += t2 - t1; t[2] += t3 - t2; t[3] += t4 - t3; t[4] += t5 - t4;
  }
  if (tid == 0) for (int i = 0; i < 5; ++i) prof[g * 8 + i] = t[i];
  if (acc == 12345.678) prof[0] = 0;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* zpart; unsigned* tw; unsigned* ctr; long long* prof;
  int n = 4096;
  cudaMalloc(&zpart, (size_t)sms * n * 8); cudaMalloc(&tw, 4096); cudaMalloc(&ctr, 4); cudaMalloc(&prof, sms * 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int rounds = 1000, T = 384;
  long long hp[148 * 8];
  auto run = [&](void* f, const char* name, int nn) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(ctr, 0, 4);
      void* args[] = {&zpart, &tw, &ctr, &nn, &rounds, &prof};
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel(f, sms, T, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) {
        cudaMemcpy(hp, prof, sms * 64, cudaMemcpyDeviceToHost);
        double s[5] = {0};
        for (int g = 0; g < sms; ++g) for (int i = 0; i < 5; ++i) s[i] += hp[g * 8 + i] / (double)sms / rounds;
        printf("%-28s n=%d %.3f us/pass | cyc: write %.0f bar1 %.0f reduce %.0f bar2 %.0f read %.0f (%s)\n", name, nn, ms * 1e3 / rounds, s[0], s[1], s[2], s[3], s[4], cudaGetErrorString(e));
        fflush(stdout);
      }
    }
  };
  run((void*)k<0, 0>, "barriers only", 4096);
  run((void*)k<1, 0>, "write + barriers", 4096);
  run((void*)k<1, 1>, "write + reduce + barriers", 4096);
  run((void*)k<1, 1>, "write + reduce + barriers", 1024);
  return 0;
}
