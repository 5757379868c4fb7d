// Per-pass exchange protocol microbenchmark (no compute): G CTAs each pass
//  (1) publish a slot {epoch, c}; every CTA gathers all G slots;
//  (2) owner CTAs publish Q tagged 64-bit words; every CTA gathers all Q words.
#include <cstdio>
#include <cuda_runtime.h>
struct Slot { unsigned epoch; unsigned pad; double c[2]; double n[2]; double pad2[3]; };
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned long long ld_rlx64(const unsigned long long* p) { unsigned long long v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ void st_rlx64(unsigned long long* p, unsigned long long v) { asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory"); }

// MODE bits: 1 = relaxed polling + one fence (else acquire per poll); 2 = nanosleep backoff;
//            4 = slot stride 128B (else 32B); 8 = only warp 0 polls t words; 16 = skip t exchange
template <int MODE>
__global__ void k(Slot* slots, unsigned long long* tw, int Q, int rounds, double* out) {
  __shared__ double red[32];
  __shared__ unsigned tws[1024];
  const int g = blockIdx.x, G = gridDim.x, tid = threadIdx.x, T = blockDim.x;
  const int stride = (MODE & 4) ? 2 : 1;  // in Slots (64B)
  double acc = 0;
  for (int P = 0; P < rounds; ++P) {
    __syncthreads();
    if (tid == 0) { Slot* my = slots + g * stride; __stcg(&my->c[P & 1], (double)g); st_rel(&my->epoch, P + 1); }
    double cs = 0;
    for (int i = tid; i < G; i += T) {
      const Slot* s = slots + i * stride;
      if (MODE & 1) {
        while ((int)(ld_rlx(&s->epoch) - (unsigned)(P + 1)) < 0) { if (MODE & 2) __nanosleep(64); }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else {
        while ((int)(ld_acq(&s->epoch) - (unsigned)(P + 1)) < 0) { if (MODE & 2) __nanosleep(64); }
      }
      cs += __ldcg(&s->c[P & 1]);
    }
    if ((tid & 31) == 0) red[tid >> 5] = cs;
    __syncthreads();
    if (!(MODE & 16)) {
      for (int q = g; q < Q; q += G) if (tid == 0) st_rlx64(tw + (P & 1) * 1024 + q, ((unsigned long long)(P + 1) << 32) | (unsigned)(q * 7 + P));
      if (!(MODE & 8) || tid < 32) {
        const int TT = (MODE & 8) ? 32 : T;
        for (int i = tid; i < Q; i += TT) {
          unsigned long long x;
          do { x = ld_rlx64(tw + (P & 1) * 1024 + i); if ((MODE & 2) && (int)((unsigned)(x >> 32) - (unsigned)(P + 1)) < 0) __nanosleep(64); } while ((int)((unsigned)(x >> 32) - (unsigned)(P + 1)) < 0);
          tws[i] = (unsigned)x;
        }
      }
      __syncthreads();
      acc += tws[tid % Q];
    }
    acc += red[0];
  }
  out[g * T + tid] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  Slot* slots; unsigned long long* tw; double* out;
  cudaMalloc(&slots, sms * 4 * sizeof(Slot)); cudaMalloc(&tw, 8 * 4096 * 2); cudaMalloc(&out, 8 * sms * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int rounds = 2000, Q = 128, T = 384;
  auto run = [&](void* f, const char* name) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(slots, 0, sms * 4 * sizeof(Slot)); cudaMemset(tw, 0, 8 * 4096 * 2);
      void* args[] = {&slots, &tw, &Q, &rounds, &out};
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel(f, sms, T, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) { printf("%-40s %.3f us per pass (%s)\n", name, ms * 1e3 / rounds, cudaGetErrorString(e)); fflush(stdout); }
    }
  };
  run((void*)k<0>, "acquire polls, 32B slots, all threads");
  run((void*)k<1>, "relaxed+fence");
  run((void*)k<3>, "relaxed+fence+sleep");
  run((void*)k<5>, "relaxed+fence, 128B-ish slots");
  run((void*)k<7>, "relaxed+fence+sleep, 128B-ish slots");
  run((void*)k<9>, "relaxed+fence, warp0 polls t");
  run((void*)k<13>, "relaxed+fence, 128B, warp0 polls t");
  run((void*)k<15>, "relaxed+fence+sleep, 128B, warp0 t");
  run((void*)k<17>, "slots only (relaxed+fence)");
  run((void*)k<21>, "slots only (relaxed+fence, 128B)");
  run((void*)k<16>, "slots only (acquire)");
  return 0;
}
