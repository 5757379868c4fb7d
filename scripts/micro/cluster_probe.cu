// Can the persistent kernel run as clusters? Max co-resident clusters of size 2/4/8
// for a 288-thread CTA with ~221 KB of dynamic shared memory, and does a cooperative
// launch with a cluster dimension succeed (grid barrier + cluster barrier round trip).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k(unsigned* bar, int* out) {
  extern __shared__ unsigned char smem[];
  cg::cluster_group cl = cg::this_cluster();
  unsigned sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  smem[threadIdx.x] = 1;
  cl.sync();
  if (threadIdx.x == 0) {
    atomicAdd(bar, 1u);
    while (atomicAdd(bar, 0u) < gridDim.x) {}
    out[blockIdx.x] = sm * 16 + cl.block_rank();
  }
}
int main() {
  size_t smem = 221 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  printf("SMs %d\n", prop.multiProcessorCount);
  for (int cs : {1, 2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 8); cfg.blockDim = dim3(288); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int nc = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k, &cfg);
    printf("cluster %d: max active clusters %d (%s) -> %d CTAs\n", cs, nc, cudaGetErrorString(e), nc * cs);
  }
  for (int cs : {2, 4}) {
    int nc = 0;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(288); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
    cfg.attrs = at; cfg.numAttrs = 1; cfg.gridDim = dim3(cs);
    cudaOccupancyMaxActiveClusters(&nc, k, &cfg);
    cfg.numAttrs = 2; cfg.gridDim = dim3(nc * cs);
    unsigned* bar; int* out; cudaMalloc(&bar, 4); cudaMalloc(&out, 4096); cudaMemset(bar, 0, 4);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, bar, out);
    cudaError_t e2 = cudaDeviceSynchronize();
    printf("cooperative cluster %d launch of %d CTAs: %s / %s\n", cs, nc * cs, cudaGetErrorString(e), cudaGetErrorString(e2));
    cudaFree(bar); cudaFree(out);
  }
  return 0;
}
