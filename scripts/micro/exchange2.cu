// Full per-pass exchange with real volumes: G CTAs x n-column f64 partials.
//  A: counter barrier -> owners reduce 32-col slices -> counter barrier -> all read t words
//  B: int64 fixed-point red.add of partials into z[P%3] -> counter barrier -> all read z, sign
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void bar_arrive(unsigned* c) { asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(c) : "memory"); }
template <int SLEEP>
__device__ __forceinline__ void bar_wait(unsigned* c, unsigned target) {
  while ((int)(ld_rlx(c) - target) < 0) { if (SLEEP) __nanosleep(SLEEP); }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
template <int SLEEP>
__global__ void protoA(double* zpart, unsigned* tw, unsigned* ctr, int n, int rounds, double* out) {
  __shared__ double seg[12][32];
  __shared__ unsigned tws[256];
  const int g = blockIdx.x, G = gridDim.x, tid = threadIdx.x, T = blockDim.x, W = T / 32, lane = tid & 31, warp = tid >> 5;
  const int Q = n / 32;
  unsigned ep = 0; double acc = 0;
  for (int P = 0; P < rounds; ++P) {
    for (int c = tid; c < n; c += T) __stcg(zpart + (size_t)g * n + c, (double)((c * 31 + g * 7 + P) % 97) - 48.0);
    __syncthreads();
    if (tid == 0) { ++ep; bar_arrive(ctr); bar_wait<SLEEP>(ctr, ep * G); }
    __syncthreads();
    for (int q = g; q < Q; q += G) {
      const int gs = warp * G / W, ge = (warp + 1) * G / W;
      double a = 0; for (int gg = gs; gg < ge; ++gg) a += __ldcg(zpart + (size_t)gg * n + q * 32 + lane);
      seg[warp][lane] = a; __syncthreads();
      if (warp == 0) { double z = 0; for (int w = 0; w < W; ++w) z += seg[w][lane]; unsigned b = __ballot_sync(~0u, z < 0); if (lane == 0) __stcg(tw + (P & 1) * 256 + q, b); }
      __syncthreads();
    }
    if (tid == 0) { ++ep; bar_arrive(ctr); bar_wait<SLEEP>(ctr, ep * G); }
    __syncthreads();
    for (int i = tid; i < Q; i += T) tws[i] = __ldcg(tw + (P & 1) * 256 + i);
    __syncthreads();
    acc += tws[tid % Q];
  }
  out[g * T + tid] = acc;
}
template <int SLEEP>
__global__ void protoB(unsigned long long* z3, unsigned* ctr, int n, int rounds, double* out) {
  __shared__ unsigned tws[256];
  const int g = blockIdx.x, G = gridDim.x, tid = threadIdx.x, T = blockDim.x;
  unsigned ep = 0; double acc = 0;
  for (int P = 0; P < rounds; ++P) {
    unsigned long long* zb = z3 + (size_t)(P % 3) * n;
    unsigned long long* zz = z3 + (size_t)((P + 1) % 3) * n;
    for (int c = tid; c < n; c += T) {
      const double v = (double)((c * 31 + g * 7 + P) % 97) - 48.0;
      const long long q = __double2ll_rn(v * 0x1p40);
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(zb + c), "l"((unsigned long long)q) : "memory");
    }
    for (int c = g * (n / G) + tid; c < (g + 1) * (n / G) + (g == G - 1 ? n % G : 0); c += T) zz[c] = 0ull;
    __syncthreads();
    if (tid == 0) { ++ep; bar_arrive(ctr); bar_wait<SLEEP>(ctr, ep * G); }
    __syncthreads();
    for (int w = tid; w < n / 32; w += T) {
      unsigned b = 0;
      for (int k = 0; k < 32; ++k) b |= ((long long)__ldcg(zb + w * 32 + k) < 0 ? 1u : 0u) << k;
      tws[w] = b;
    }
    __syncthreads();
    acc += tws[tid % (n / 32)];
  }
  out[g * T + tid] = acc;
}
__global__ void redonly(unsigned long long* z, int n, int rounds) {
  for (int P = 0; P < rounds; ++P)
    for (int c = threadIdx.x; c < n; c += blockDim.x)
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" :: "l"(z + c), "l"((unsigned long long)(blockIdx.x + P)) : "memory");
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* zpart; unsigned* tw; unsigned* ctr; unsigned long long* z3; double* out;
  const int n = 4096;
  cudaMalloc(&zpart, (size_t)sms * n * 8); cudaMalloc(&tw, 4096); cudaMalloc(&ctr, 4); cudaMalloc(&z3, 3 * n * 8); cudaMalloc(&out, sms * 1024 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int rounds = 1000, T = 384; int nn = n;
  auto time = [&](void* f, void** args, const char* name) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(ctr, 0, 4); cudaMemset(z3, 0, 3 * n * 8);
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel(f, sms, T, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) { printf("%-44s %.3f us per pass (%s)\n", name, ms * 1e3 / rounds, cudaGetErrorString(e)); fflush(stdout); }
    }
  };
  { void* args[] = {&zpart, &tw, &ctr, &nn, &rounds, &out}; time((void*)protoA<0>, args, "A: 2 barriers + owner reduce (spin)"); }
  { void* args[] = {&zpart, &tw, &ctr, &nn, &rounds, &out}; time((void*)protoA<64>, args, "A: 2 barriers + owner reduce (sleep64)"); }
  { void* args[] = {&z3, &ctr, &nn, &rounds, &out}; time((void*)protoB<0>, args, "B: int64 red + 1 barrier (spin)"); }
  { void* args[] = {&z3, &ctr, &nn, &rounds, &out}; time((void*)protoB<64>, args, "B: int64 red + 1 barrier (sleep64)"); }
  { void* args[] = {&z3, &nn, &rounds}; time((void*)redonly, args, "red.add.u64 only (148 x 4096 per pass)"); }
  return 0;
}
