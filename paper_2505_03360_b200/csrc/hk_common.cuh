// hk_common.cuh — shared device helpers for the hykin B200 collision path.
//
// Register-resident complex FFTs (one pencil per thread, fully unrolled so
// every index is a compile-time constant and the pencil lives in registers),
// complex arithmetic on double2, and cluster/DSMEM helpers.  fp64 only: the
// reference path is double precision end to end (inc/spectral.hpp:15-33).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hk {

namespace cg = cooperative_groups;

// e^{-2 pi i k / 64}, k = 0..31, correctly rounded (generated with 50-digit
// arithmetic).  Radix-2 stages of an N-point transform (N | 64) index it with
// stride 64/N.
__device__ __constant__ double2 c_tw64[32] = {
    {1.0, 0.0},
    {0.9951847266721969, -0.0980171403295606},
    {0.9807852804032304, -0.19509032201612828},
    {0.9569403357322088, -0.2902846772544624},
    {0.9238795325112867, -0.3826834323650898},
    {0.881921264348355, -0.47139673682599764},
    {0.8314696123025452, -0.5555702330196022},
    {0.773010453362737, -0.6343932841636455},
    {0.7071067811865476, -0.7071067811865476},
    {0.6343932841636455, -0.773010453362737},
    {0.5555702330196022, -0.8314696123025452},
    {0.47139673682599764, -0.881921264348355},
    {0.3826834323650898, -0.9238795325112867},
    {0.2902846772544624, -0.9569403357322088},
    {0.19509032201612828, -0.9807852804032304},
    {0.0980171403295606, -0.9951847266721969},
    {0.0, -1.0},
    {-0.0980171403295606, -0.9951847266721969},
    {-0.19509032201612828, -0.9807852804032304},
    {-0.2902846772544624, -0.9569403357322088},
    {-0.3826834323650898, -0.9238795325112867},
    {-0.47139673682599764, -0.881921264348355},
    {-0.5555702330196022, -0.8314696123025452},
    {-0.6343932841636455, -0.773010453362737},
    {-0.7071067811865476, -0.7071067811865476},
    {-0.773010453362737, -0.6343932841636455},
    {-0.8314696123025452, -0.5555702330196022},
    {-0.881921264348355, -0.47139673682599764},
    {-0.9238795325112867, -0.3826834323650898},
    {-0.9569403357322088, -0.2902846772544624},
    {-0.9807852804032304, -0.19509032201612828},
    {-0.9951847266721969, -0.0980171403295606}};

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }

template <int N>
__host__ __device__ constexpr int bitrev(int i) {
    int r = 0;
    for (int b = 0; b < ilog2c(N); ++b) r |= ((i >> b) & 1) << (ilog2c(N) - 1 - b);
    return r;
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// d * w_N^{k} with w = e^{-2 pi i / N} (forward) or its conjugate (inverse).
// k is a compile-time constant after unrolling; trivial twiddles fold away.
template <int N, bool INV>
__device__ __forceinline__ double2 twiddle(double2 d, int k) {
    if (k == 0) return d;
    if (4 * k == N) {  // w^{N/4} = -i (forward) / +i (inverse)
        return INV ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);
    }
    double2 w = c_tw64[k * (64 / N)];
    if (INV) w.y = -w.y;
    return cmul(d, w);
}

// In-register radix-2 decimation-in-frequency transform of N complex values,
// natural order in and out (the bit-reversal is a compile-time renaming).
// Unnormalised: forward = sum x_j e^{-2 pi i jk/N} (FFTW_FORWARD), inverse
// = sum x_j e^{+2 pi i jk/N} (FFTW_BACKWARD), as used by src/fft.cpp:49-81.
template <int N, bool INV>
__device__ __forceinline__ void fft_reg(double2 (&x)[N]) {
#pragma unroll
    for (int len = N; len >= 2; len >>= 1) {
        const int half = len >> 1;
#pragma unroll
        for (int i = 0; i < N; i += len) {
#pragma unroll
            for (int j = 0; j < half; ++j) {
                const double2 a = x[i + j], b = x[i + j + half];
                x[i + j] = cadd(a, b);
                x[i + j + half] = twiddle<N, INV>(csub(a, b), j * (N / len));
            }
        }
    }
    double2 y[N];
#pragma unroll
    for (int i = 0; i < N; ++i) y[bitrev<N>(i)] = x[i];
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = y[i];
}

// Cluster barrier split into arrive (release) / wait (acquire) so that
// independent work can run between the two (PTX barrier.cluster).
__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_id_x() {
    unsigned r;
    asm volatile("mov.u32 %0, %%clusterid.x;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned n_clusters_x() {
    unsigned r;
    asm volatile("mov.u32 %0, %%nclusterid.x;\n" : "=r"(r));
    return r;
}

// Address of `p` (a pointer into this CTA's shared memory) in the shared
// memory of cluster rank `rank`, as a generic pointer (DSMEM window).
template <typename T>
__device__ __forceinline__ T* dsmem_ptr(T* p, unsigned rank) {
    return cg::this_cluster().map_shared_rank(p, rank);
}

// Non-negative double max via its ordered bit pattern.
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

}  // namespace hk
