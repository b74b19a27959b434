// Prints cudaOccupancyMaxActiveClusters for cluster sizes 1..16 with a 128-thread, 68 KB kernel.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(128, 2) dummy(int* p) { if (p) p[threadIdx.x] = 0; }
int main() {
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int pol = 0; pol < 3; ++pol)
  for (int c : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {}; cudaLaunchAttribute a[2];
    a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = c; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    a[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference; a[1].val.clusterSchedulingPolicyPreference = (cudaClusterSchedulingPolicy)pol;
    cfg.gridDim = dim3(c * 64); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 68000; cfg.attrs = a; cfg.numAttrs = 2;
    int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
    int n2=-1; cfg.dynamicSmemBytes = 200000; cudaOccupancyMaxActiveClusters(&n2, dummy, &cfg);
    printf("policy %d cluster %2d: max active clusters %d (CTAs %d) [1 CTA/SM smem: %d] %s\n", pol, c, n, n * c, n2, cudaGetErrorString(e));
  }
  return 0;
}
