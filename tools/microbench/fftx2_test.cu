// Unit test of the split-pencil transforms against fft_reg<32>.
#include <cstdio>
#include "../../paper_2505_03360_b200/csrc/hk_common.cuh"
using namespace hk;
__global__ void k(const double2* in, double* err) {
  const int lane = threadIdx.x & 31, p = lane & 15, h = lane >> 4;
  const double2* x = in + (blockIdx.x * 16 + p) * 32;
  double2 ref[32];
  for (int i = 0; i < 32; ++i) ref[i] = x[i];
  fft_reg<32, false>(ref);
  double2 v[16];
  for (int m = 0; m < 16; ++m) v[m] = x[2 * m + h];
  fftx2_dit<false>(v, h);
  double e = 0;
  for (int j = 0; j < 8; ++j) {
    e = fmax(e, fabs(v[j].x - ref[8 * h + j].x) + fabs(v[j].y - ref[8 * h + j].y));
    e = fmax(e, fabs(v[8 + j].x - ref[16 + 8 * h + j].x) + fabs(v[8 + j].y - ref[16 + 8 * h + j].y));
  }
  double2 u[16];
  for (int j = 0; j < 8; ++j) { u[j] = x[8 * h + j]; u[8 + j] = x[16 + 8 * h + j]; }
  fftx2_dif<false>(u, h);
  for (int m = 0; m < 16; ++m) e = fmax(e, fabs(u[m].x - ref[2 * m + h].x) + fabs(u[m].y - ref[2 * m + h].y));
  // inverse round trip: DIT inverse of the parity-split forward output returns 32 x (index halves)
  fftx2_dit<true>(u, h);
  for (int j = 0; j < 8; ++j) {
    e = fmax(e, fabs(u[j].x / 32 - x[8 * h + j].x) + fabs(u[j].y / 32 - x[8 * h + j].y));
    e = fmax(e, fabs(u[8 + j].x / 32 - x[16 + 8 * h + j].x) + fabs(u[8 + j].y / 32 - x[16 + 8 * h + j].y));
  }
  atomicMax((unsigned long long*)err, (unsigned long long)__double_as_longlong(e));
}
int main() {
  const int nb = 64, n = nb * 16 * 32;
  double2* h_in = new double2[n];
  for (int i = 0; i < n; ++i) h_in[i] = make_double2(sin(0.37 * i) + 0.1 * (i % 7), cos(1.3 * i) - 0.05 * (i % 5));
  double2* d_in; double* d_err; cudaMalloc(&d_in, n * 16); cudaMalloc(&d_err, 8); cudaMemset(d_err, 0, 8);
  cudaMemcpy(d_in, h_in, n * 16, cudaMemcpyHostToDevice);
  k<<<nb, 32>>>(d_in, d_err);
  double e = -1; cudaError_t st = cudaDeviceSynchronize(); cudaMemcpy(&e, d_err, 8, cudaMemcpyDeviceToHost);
  printf("{\"fftx2\": \"%s\", \"max_err\": %.3e}\n", cudaGetErrorString(st), e);
  return (st == cudaSuccess && e < 1e-12) ? 0 : 1;
}
