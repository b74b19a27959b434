// hk_weights.cu — device construction of the spectral weight tables.
//
// Replaces precompute_kernel (src/spectral.cpp:53-112).  Two steps:
//  1. closed_form_raw_tables: alpha_d, alpha'_d in the reference layout
//     [a1*a2][i1][i2][i3] and loss_diag, from the closed forms of
//     hs_radial_transform / hs_planar_transform (src/spectral.cpp:43-51):
//        phi(s) = 4 [ r sin(rs)/s - 2 sin^2(rs/2)/s^2 ],  phi(0) = 2 r^2
//        psi(t) = 16 sin^2(rt/2) / t^2,                    psi(0) = 4 r^2
//     (the adaptive GK15 quadrature of src/quadrature.cpp agrees to ~1e-14).
//  2. build_kernel_tables: from raw tables (closed form, or the reference's
//     own tables uploaded verbatim) build the device layouts:
//        exact  alpha / alpha_p / loss   [entry][i1][i3][i2]
//        fast   (alpha_s, alpha'_s)      Hermitian-symmetrised, entry md = (loss_s, 0);
//                                         at n = 64 [entry][i1][i2 / 16][i3][i2 % 16] (warp blocks)
//        nyquist alpha_a, alpha'_a  antisymmetric parts on the three Nyquist planes
//                                   (signed: the guard takes |.|, the correction kernel the values).
#include <cmath>

#include "hk_common.cuh"
#include "hk_internal.h"

namespace hk {

namespace {

__device__ __forceinline__ int freq(int idx, int n) { return idx < n / 2 ? idx : idx - n; }  // inc/fft.hpp:69

__device__ double radial_closed(double s, double r) {
    if (s == 0.0) return 2.0 * r * r;
    const double h = sin(0.5 * r * s);
    return 4.0 * (r * sin(r * s) / s - 2.0 * h * h / (s * s));
}

__device__ double planar_closed(double t, double r) {
    if (t == 0.0) return 4.0 * r * r;
    const double h = sin(0.5 * r * t);
    return 16.0 * h * h / (t * t);
}

// Raw tables in the reference order d = p*a2 + q, idx = (i1*n + i2)*n + i3.
__global__ void raw_tables_kernel(int n, int a1, int a2, double r, double weight,
                                  double* __restrict__ alpha, double* __restrict__ alpha_p,
                                  double* __restrict__ loss) {
    const int64_t total = (int64_t)n * n * n;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const int i3 = idx % n, i2 = (idx / n) % n, i1 = idx / ((int64_t)n * n);
    const double l1 = freq(i1, n), l2 = freq(i2, n), l3 = freq(i3, n);
    // No FMA contraction: mirror the reference's rounding (src/spectral.cpp:100-102).
    const double l2norm = __dadd_rn(__dadd_rn(__dmul_rn(l1, l1), __dmul_rn(l2, l2)), __dmul_rn(l3, l3));
    double acc = 0.0;
    for (int p = 0; p < a1; ++p) {
        const double theta = p * M_PI / a1;
        for (int q = 0; q < a2; ++q) {
            const double phi = q * M_PI / a2;
            const double e0 = __dmul_rn(sin(theta), cos(phi));
            const double e1 = __dmul_rn(sin(theta), sin(phi));
            const double e2 = cos(theta);
            const double ldote = __dadd_rn(__dadd_rn(__dmul_rn(l1, e0), __dmul_rn(l2, e1)), __dmul_rn(l3, e2));
            const double perp2 = fmax(0.0, __dadd_rn(l2norm, -__dmul_rn(ldote, ldote)));
            const double a = radial_closed(ldote, r);
            const double ap = planar_closed(sqrt(perp2), r);
            const int d = p * a2 + q;
            alpha[(int64_t)d * total + idx] = a;
            alpha_p[(int64_t)d * total + idx] = ap;
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(weight, a), ap));  // src/spectral.cpp:105
        }
    }
    loss[idx] = acc;
}

__device__ __forceinline__ int entry_to_dir(int e, int a2) { return e == 0 ? 0 : a2 + (e - 1); }

// One thread per mode (i1, i2, i3); writes every entry of the device layouts.
__global__ void layout_kernel(int n, int a2, int md, const double* __restrict__ ra,
                              const double* __restrict__ rap, const double* __restrict__ rl,
                              double* __restrict__ alpha, double* __restrict__ alpha_p,
                              double* __restrict__ loss, double2* __restrict__ wfast,
                              double* __restrict__ abs_a, double* __restrict__ abs_ap) {
    const int64_t total = (int64_t)n * n * n;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const int i3 = idx % n, i2 = (idx / n) % n, i1 = idx / ((int64_t)n * n);
    const int m1 = (n - i1) % n, m2 = (n - i2) % n, m3 = (n - i3) % n;
    const int64_t midx = ((int64_t)m1 * n + m2) * n + m3;
    const int64_t dev = ((int64_t)i1 * n + i3) * n + i2;  // [i1][i3][i2]
    // fast table at n = 64: [i1][i2 / 16][i3][i2 % 16], so the 16 pencils of one
    // producer warp of coll64_w12_kernel are one contiguous 16 KiB block (one bulk copy)
    const int64_t fdev = n == 64 ? (((int64_t)i1 * 4 + (i2 >> 4)) * n + i3) * 16 + (i2 & 15) : dev;
    const int h = n / 2;
    const int64_t nn = (int64_t)n * n;
    for (int e = 0; e < md; ++e) {
        const int d = entry_to_dir(e, a2);
        const double a = ra[(int64_t)d * total + idx], am = ra[(int64_t)d * total + midx];
        const double ap = rap[(int64_t)d * total + idx], apm = rap[(int64_t)d * total + midx];
        alpha[(int64_t)e * total + dev] = a;
        alpha_p[(int64_t)e * total + dev] = ap;
        wfast[(int64_t)e * total + fdev] = make_double2(0.5 * (a + am), 0.5 * (ap + apm));
        const double aa = 0.5 * (a - am), aap = 0.5 * (ap - apm);  // signed antisymmetric parts
        double* pa = abs_a + (int64_t)e * 3 * nn;
        double* pap = abs_ap + (int64_t)e * 3 * nn;
        // Nyquist planes, each S point counted once (plane 0, then 1, then 2).
        if (i1 == h) {
            pa[0 * nn + i2 * n + i3] = aa;
            pap[0 * nn + i2 * n + i3] = aap;
        } else if (i2 == h) {
            pa[1 * nn + i1 * n + i3] = aa;
            pap[1 * nn + i1 * n + i3] = aap;
        } else if (i3 == h) {
            pa[2 * nn + i1 * n + i2] = aa;
            pap[2 * nn + i1 * n + i2] = aap;
        }
    }
    loss[dev] = rl[idx];
    wfast[(int64_t)md * total + fdev] = make_double2(0.5 * (rl[idx] + rl[midx]), 0.0);
}

}  // namespace

int closed_form_raw_tables(hk_ctx ctx, hk_kernel k, double* ra, double* rap, double* rl) {
    const int64_t total = (int64_t)k->n * k->n * k->n;
    const int threads = 256;
    const int blocks = int((total + threads - 1) / threads);
    raw_tables_kernel<<<blocks, threads, 0, ctx->stream>>>(k->n, k->a1, k->a2, k->r, k->weight, ra,
                                                          rap, rl);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "raw_tables_kernel");
}

int build_kernel_tables(hk_ctx ctx, hk_kernel k, const double* ra, const double* rap,
                        const double* rl) {
    const int n = k->n;
    const int64_t total = (int64_t)n * n * n;
    const size_t nn3 = size_t(3) * n * n;
    int st;
    if ((st = check_cuda(ctx, cudaMalloc(&k->alpha, sizeof(double) * total * k->md), "alloc alpha"))) return st;
    if ((st = check_cuda(ctx, cudaMalloc(&k->alpha_p, sizeof(double) * total * k->md), "alloc alpha_p"))) return st;
    if ((st = check_cuda(ctx, cudaMalloc(&k->loss, sizeof(double) * total), "alloc loss"))) return st;
    if ((st = check_cuda(ctx, cudaMalloc(&k->wfast, sizeof(double2) * total * (k->md + 1)), "alloc wfast"))) return st;
    if ((st = check_cuda(ctx, cudaMalloc(&k->abs_a, sizeof(double) * nn3 * k->md), "alloc abs_a"))) return st;
    if ((st = check_cuda(ctx, cudaMalloc(&k->abs_ap, sizeof(double) * nn3 * k->md), "alloc abs_ap"))) return st;
    cudaMemsetAsync(k->abs_a, 0, sizeof(double) * nn3 * k->md, ctx->stream);
    cudaMemsetAsync(k->abs_ap, 0, sizeof(double) * nn3 * k->md, ctx->stream);
    const int threads = 256;
    const int blocks = int((total + threads - 1) / threads);
    layout_kernel<<<blocks, threads, 0, ctx->stream>>>(n, k->a2, k->md, ra, rap, rl, k->alpha,
                                                      k->alpha_p, k->loss, k->wfast, k->abs_a,
                                                      k->abs_ap);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "layout_kernel");
}

}  // namespace hk
