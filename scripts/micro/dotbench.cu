// Isolated dot_pass benchmark: rows resident in SMEM, no producer, no grid sync.
#include "../../paper_2410_01799_b200/csrc/sweep.cu"
#include <cstdio>
#include <vector>
namespace scb {
template <int NW, int VPT, int RG, int TWO>
__global__ void __launch_bounds__((NW + 1) * 32, 1) dotbench(int rows, int n, int passes, long long* cyc, double* zout, int wmul, unsigned long long* tprof) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int pitch = (n + 31) / 32 * 32;
  const size_t rowB = pitch * 4;
  const int Q = pitch / 32;
  const Layout L = make_layout(rowB, 0, rows, RG, NW, rows, Q, 1, (rows + 31) / 32);
  const int tid = threadIdx.x;
  float* rowsmem = reinterpret_cast<float*>(smem + L.res);
  for (int i = tid; i < rows * pitch; i += blockDim.x) rowsmem[i] = ((i * 7919) % 1000) * 0.001f - 0.5f;
  uint32_t* tws = reinterpret_cast<uint32_t*>(smem + L.tws);
  for (int i = tid; i < Q; i += blockDim.x) tws[i] = 0x5a5a5a5au ^ (i * 2654435761u);
  unsigned long long* ring = reinterpret_cast<unsigned long long*>(smem + L.ring);
  if (tid == 0) {
    for (int s = 0; s < kRing; ++s) mbar_init(&ring[s], NW);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t* sb = reinterpret_cast<uint32_t*>(smem + L.sb);
  for (int i = tid; i < 3 * ((rows + 31) / 32); i += blockDim.x) sb[i] = 0;
  __syncthreads();
  if (tid >= NW * 32) return;
  DotArgs a;
  a.res = L.res; a.stage = L.stage; a.full = 0; a.empty = 0; a.ring = L.ring; a.rred = L.rred; a.yrow = L.yrow;
  a.s_nxt = L.sb; a.tws = L.tws; a.zrow = zout + (size_t)blockIdx.x * pitch; a.errp = nullptr;
  a.rowB = rowB; a.rows_g = rows; a.nres = rows; a.D = 0; a.NV = pitch / 4; a.sslot = 0; a.sph = 0;
  unsigned gcount = 0;
  const long long t0 = clock64();
  for (int P = 0; P < passes; ++P) {
    a.P = P; a.gcount = gcount; a.wmul = wmul; a.ypart = L.ypart; a.prof = nullptr;
#ifdef SCB_TIMING
    a.tprof = tprof;
#endif
    if (TWO) dot_pass_2ph<float, NW, VPT>(a); else dot_pass<float, NW, VPT, RG>(a);
    gcount += (rows + RG - 1) / RG;
    asm volatile("bar.sync 1, %0;" :: "r"(NW * 32));
  }
  if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
}
}  // namespace scb
template <int NW, int VPT, int RG, int TWO = 0>
void run(int rows, int n, const char* name) {
  using namespace scb;
  int pitch = (n + 31) / 32 * 32;
  size_t rowB = pitch * 4;
  Layout L = make_layout(rowB, 0, rows, RG, NW, rows, pitch / 32, 1, (rows + 31) / 32);
  auto f = dotbench<NW, VPT, RG, TWO>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  long long* cyc; double* z; cudaMalloc(&cyc, 8 * 148); cudaMalloc(&z, 8 * 148 * (size_t)pitch);
  int passes = 200;
  unsigned long long* tp; cudaMalloc(&tp, 148 * 32 * 8 * 8); cudaMemset(tp, 0, 148 * 32 * 8 * 8);
  f<<<148, (NW + 1) * 32, L.total>>>(rows, n, passes, cyc, z, 1 << 29, tp);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(148); cudaMemcpy(h.data(), cyc, 8 * 148, cudaMemcpyDeviceToHost);
  double avg = 0; for (auto v : h) avg += v; avg /= 148.0 * passes;
#ifdef SCB_TIMING
  { std::vector<unsigned long long> t(148 * 32 * 8); cudaMemcpy(t.data(), tp, t.size() * 8, cudaMemcpyDeviceToHost);
    const char* nm[8] = {"rows_of", "combine", "widen+dot(+ld)", "reduce", "zupd(+ld)", "sts", "barrier", "rec+rel"};
    for (int w : {0, 4, 7}) { printf("warp %d:", w); double tot = 0;
      for (int k = 0; k < 8; ++k) { double c = 0; for (int b = 0; b < 148; ++b) c += t[(b * 32 + w) * 8 + k]; c /= 148.0 * passes * rows; tot += c; printf(" %s=%.0f", nm[k], c); }
      printf(" | sum=%.0f cycles/row\n", tot); } }
#endif
  printf("%-12s rows=%3d n=%5d: %8.0f cycles/pass  %6.0f cycles/row  %.2f elem/clk/SM  (%s)\n", name, rows, n, avg, avg / rows,
         rows * (double)n / avg, cudaGetErrorString(e));
}
int main(int argc, char** argv) {
  if (argc > 1) { run<8, 4, 1, 1>(12, 4096, "2ph 8,4"); return 0; }
  run<8, 4, 1, 1>(12, 4096, "2ph 8,4");
  run<8, 4, 1, 1>(24, 4096, "2ph 8,4");
  run<16, 2, 1, 1>(12, 4096, "2ph 16,2");
  run<8, 4, 1>(7, 4096, "8,4,1");
  run<8, 4, 1>(12, 4096, "8,4,1");
  run<8, 1, 4>(7, 1024, "8,1,4");
  run<8, 4, 2>(12, 4096, "8,4,2");
  run<16, 2, 1>(12, 4096, "16,2,1");
  run<8, 2, 2>(12, 2048, "8,2,2");
  return 0;
}
