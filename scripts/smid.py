"""Which SM does each CTA of the persistent kernel land on? (cooperative launch,
one CTA per SM)  Prints CTA -> SM id via a tiny probe kernel with the same grid."""
import torch
src = r'''
extern "C" __global__ void probe(int* out) {
  unsigned sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  if (threadIdx.x == 0) out[blockIdx.x] = sm;
}'''
from torch.utils.cpp_extension import load_inline
