// Grid-barrier designs for 148 co-resident CTAs.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) { unsigned r; asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory"); return r; }
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) { asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ void fence_acq() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// MODE 0: flat counter, relaxed poll + fence
// MODE 1: 2-level tree: group counters (GS CTAs), last arriver bumps root; all poll root
// MODE 2: 2-level tree, last arriver at root writes release flag (epoch); all poll flag
// MODE 3: flat counter via atom with return; last arriver writes flag; others poll flag
template <int MODE, int GS>
__global__ void k(unsigned* mem, int rounds, long long* out) {
  unsigned* root = mem;            // line 0
  unsigned* flag = mem + 32;       // line 1
  unsigned* grp = mem + 64;        // group counters, one line each
  const int g = blockIdx.x, G = gridDim.x;
  const int ng = (G + GS - 1) / GS, mg = g / GS;
  const int gsz = min(GS, G - mg * GS);
  unsigned ep = 0;
  for (int P = 0; P < rounds; ++P) {
    __syncthreads();
    if (threadIdx.x == 0) {
      ++ep;
      if (MODE == 0) {
        red_rel(root, 1);
        while ((int)(ld_rlx(root) - ep * G) < 0) {}
        fence_acq();
      } else if (MODE == 1) {
        if (atom_add_acqrel(grp + mg * 32, 1) == ep * gsz - 1) red_rel(root, 1);
        while ((int)(ld_rlx(root) - ep * ng) < 0) {}
        fence_acq();
      } else if (MODE == 2) {
        if (atom_add_acqrel(grp + mg * 32, 1) == ep * gsz - 1)
          if (atom_add_acqrel(root, 1) == ep * ng - 1) st_rel(flag, ep);
        while ((int)(ld_rlx(flag) - ep) < 0) {}
        fence_acq();
      } else if (MODE == 3) {
        if (atom_add_acqrel(root, 1) == ep * G - 1) st_rel(flag, ep);
        while ((int)(ld_rlx(flag) - ep) < 0) {}
        fence_acq();
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[g] = ep;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* mem; long long* out; cudaMalloc(&mem, 64 * 1024); cudaMalloc(&out, 8 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int rounds = 10000;
  auto run = [&](void* f, const char* name) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(mem, 0, 64 * 1024);
      void* args[] = {&mem, &rounds, &out};
      cudaEventRecord(a);
      cudaError_t e = cudaLaunchCooperativeKernel(f, sms, 384, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) { printf("%-36s %.3f us (%s)\n", name, ms * 1e3 / rounds, cudaGetErrorString(e)); fflush(stdout); }
    }
  };
  run((void*)k<0, 1>, "flat counter");
  run((void*)k<1, 8>, "tree GS=8, poll root");
  run((void*)k<1, 16>, "tree GS=16, poll root");
  run((void*)k<1, 32>, "tree GS=32, poll root");
  run((void*)k<2, 8>, "tree GS=8, flag");
  run((void*)k<2, 16>, "tree GS=16, flag");
  run((void*)k<3, 1>, "flat atom + flag");
  return 0;
}
