// TMEM round-trip check: each thread stores 64 doubles into its lane and reads them back.
#include <cstdio>
#include "../../paper_2505_03360_b200/csrc/hk_common.cuh"
using namespace hk;
__global__ void __launch_bounds__(128, 2) k(double* out, int* bad) {
  __shared__ uint32_t slot;
  const int t = threadIdx.x, w = t >> 5;
  if (w == 0) tmem_alloc(&slot, 256);
  tmem_fence_before(); __syncthreads(); tmem_fence_after();
  const uint32_t base = slot + ((uint32_t)(32 * (w & 3)) << 16);
  for (int c = 0; c < 8; ++c) {
    double v[8];
    for (int i = 0; i < 8; ++i) v[i] = blockIdx.x * 1e6 + t * 1000 + c * 8 + i + 0.25;
    tmem_st16(base + 16 * c, v);
  }
  tmem_wait_st();
  double s = 0; int nb = 0;
  for (int c = 0; c < 8; ++c) {
    double v[8];
    tmem_ld16(base + 16 * c, v);
    for (int i = 0; i < 8; ++i) { double e = blockIdx.x * 1e6 + t * 1000 + c * 8 + i + 0.25; if (v[i] != e) nb++; s += v[i]; }
  }
  atomicAdd(bad, nb);
  out[blockIdx.x * 128 + t] = s;
  tmem_fence_before(); __syncthreads(); tmem_fence_after();
  if (w == 0) tmem_dealloc(slot, 256);
}
int main() {
  double* out; int* bad; cudaMalloc(&out, 296 * 128 * 8); cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4);
  k<<<296, 128>>>(out, bad);
  cudaError_t e = cudaDeviceSynchronize();
  int hb = -1; cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  printf("{\"tmem_test\": \"%s\", \"mismatches\": %d}\n", cudaGetErrorString(e), hb);
  return 0;
}
