#include "whit_kernels.cuh"
#include <cstdio>
int main() {
  cudaFuncAttributes a;
  auto k1 = whit::whit_kernel<2, float, true, false, true>;
  auto k2 = whit::whit_kernel<2, float, true, true, true>;
  auto k3 = whit::whit_kernel<2, float, true, false, false>;
  for (auto k : {k1, k2, k3}) {
    cudaFuncGetAttributes(&a, k);
    printf("regs %d maxThreadsPerBlock %d static smem %zu local %zu\n", a.numRegs, a.maxThreadsPerBlock, a.sharedSizeBytes, a.localSizeBytes);
  }
  return 0;
}
