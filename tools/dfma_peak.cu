// fp64 FMA peak microbenchmark (roofline denominator for the collision kernel).
// Each thread runs 8 independent DFMA chains; grid = 148 SMs x 8 CTAs x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}
__global__ void dadd_loop(double* out, int iters, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 += b; x1 += b; x2 += b; x3 += b; x4 += b; x5 += b; x6 += b; x7 += b;
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  double* out; cudaMalloc(&out, 8);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * 16 * double(iters) * blocks * threads;
  float bestadd = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0); dadd_loop<<<blocks, threads>>>(out, iters, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < bestadd) bestadd = ms;
  }
  double adds = 8.0 * 16 * double(iters) * blocks * threads;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"fp64_fma_tflops\": %.3f, \"fp64_add_tops\": %.3f, \"fma_ms\": %.3f}\n",
         p.name, p.multiProcessorCount, flops / best / 1e9, adds / bestadd / 1e9, best);
  return 0;
}
