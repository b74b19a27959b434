// hk_euler.cu — Layer-0 compressible Euler solver and the layer-0 <-> layer-1
// transitions (SURVEY §8f "next" rows 1-2), sm_100a.
//
//   euler_rhs_periodic     src/euler.cpp:159-170 (euler_rhs_cell :143-157,
//                          face_flux :124-141, cweno3 :10-40, LF flux :116-121)
//   tvd_rk2_step_periodic  src/euler.cpp:172-181
//   moments_from_conserved / conserved_from_moments   src/coupling.cpp:7-22
//   convert_on_transition  src/regime.cpp:54-72 (0 -> 1: Maxwellian of the
//                          hydro state; 1 -> 0: hydro state of the moments)
// One thread per cell; compiled without FMA contraction and with the
// reference's statement order, so the results are bitwise those of the
// reference (tests/test_gpu_euler.py).  A non-positive density or pressure of
// a cell or of a reconstructed face state is the reference's positivity_error:
// the lowest such cell is reported (HK_POSITIVITY, hk_last_error).
#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "hk_cells.cuh"
#include "hk_common.cuh"
#include "hk_internal.h"

namespace hk {

namespace {

struct Prim {
    double rho, ux, uy, p;
};

__device__ __forceinline__ bool to_primitive(const double* u, double xi, Prim& q) {  // :66-82
    if (!(u[0] > 0.0)) return false;
    const double p = (xi - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
    if (!(p > 0.0)) return false;
    q.rho = u[0];
    q.p = p;
    q.ux = u[1] / u[0];
    q.uy = u[2] / u[0];
    return true;
}

__device__ __forceinline__ void cweno3_ref(double um, double uc, double up, double eps, double& left, double& right) {
    const double sl = uc - um, sr = up - uc;
    const double b = 0.5 * (up - um);
    const double c = up - 2.0 * uc + um;
    const double is_l = sl * sl, is_r = sr * sr;
    const double is_c = (13.0 / 3.0) * c * c + b * b;
    double al = 0.25 / ((eps + is_l) * (eps + is_l));
    double ac = 0.50 / ((eps + is_c) * (eps + is_c));
    double ar = 0.25 / ((eps + is_r) * (eps + is_r));
    const double inv = 1.0 / (al + ac + ar);
    al *= inv;
    ac *= inv;
    ar *= inv;
    const double pc_a = uc - c / 12.0;
    const double c0 = al * uc + ar * uc + ac * pc_a;
    const double c1 = al * sl + ar * sr + ac * b;
    const double c2 = ac * c;
    left = c0 - 0.5 * c1 + 0.25 * c2;
    right = c0 + 0.5 * c1 + 0.25 * c2;
}

__device__ __forceinline__ void to_conserved(const Prim& p, double xi, double (&u)[4]) {  // :84-91
    u[0] = p.rho;
    u[1] = p.rho * p.ux;
    u[2] = p.rho * p.uy;
    u[3] = p.p / (xi - 1.0) + 0.5 * p.rho * (p.ux * p.ux + p.uy * p.uy);
}

__device__ __forceinline__ bool euler_flux(const double (&u)[4], int axis, double xi, double (&f)[4]) {  // :95-108
    if (!(u[0] > 0.0)) return false;
    const double p = (xi - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
    if (!(p > 0.0)) return false;
    const double un = (axis == 0 ? u[1] : u[2]) / u[0];
    f[0] = u[0] * un;
    f[1] = u[1] * un;
    f[2] = u[2] * un;
    if (axis == 0) f[1] += p;
    else f[2] += p;
    f[3] = un * (u[3] + p);
    return true;
}

__device__ bool face_flux(const Prim& q0, const Prim& q1, const Prim& q2, const Prim& q3, int axis, double xi,
                          double eps, double (&out)[4]) {  // :124-141
    Prim l, r;
    double d;
    cweno3_ref(q0.rho, q1.rho, q2.rho, eps, d, l.rho);
    cweno3_ref(q0.ux, q1.ux, q2.ux, eps, d, l.ux);
    cweno3_ref(q0.uy, q1.uy, q2.uy, eps, d, l.uy);
    cweno3_ref(q0.p, q1.p, q2.p, eps, d, l.p);
    cweno3_ref(q1.rho, q2.rho, q3.rho, eps, r.rho, d);
    cweno3_ref(q1.ux, q2.ux, q3.ux, eps, r.ux, d);
    cweno3_ref(q1.uy, q2.uy, q3.uy, eps, r.uy, d);
    cweno3_ref(q1.p, q2.p, q3.p, eps, r.p, d);
    if (!(l.rho > 0.0) || !(l.p > 0.0) || !(r.rho > 0.0) || !(r.p > 0.0)) return false;
    const double ul = axis == 0 ? l.ux : l.uy, ur = axis == 0 ? r.ux : r.uy;
    const double cl = sqrt(xi * l.p / l.rho), cr = sqrt(xi * r.p / r.rho);
    const double a = fmax(fabs(ul) + cl, fabs(ur) + cr);  // max_wave_speed :110-114
    double uL[4], uR[4], fl[4], fr[4];
    to_conserved(l, xi, uL);
    to_conserved(r, xi, uR);
    if (!euler_flux(uL, axis, xi, fl) || !euler_flux(uR, axis, xi, fr)) return false;
    for (int k = 0; k < 4; ++k) out[k] = 0.5 * (fl[k] + fr[k]) - (0.5 * a) * (uR[k] - uL[k]);
    return true;
}

// rhs = -dF/dx - dG/dy on the periodic torus; *bad = lowest failing cell.
__global__ void euler_rhs_kernel(const double* __restrict__ u, int nx, int ny, double dx, double dy, double xi,
                                 double eps, double* __restrict__ out, unsigned long long* __restrict__ bad) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= (int64_t)nx * ny) return;
    const int i = (int)(c % nx), j = (int)(c / nx);
    Prim px[5], py[5];
    bool ok = true;
    for (int k = -2; k <= 2; ++k) {
        const int ii = ((i + k) % nx + nx) % nx, jj = ((j + k) % ny + ny) % ny;
        ok &= to_primitive(u + 4 * ((int64_t)j * nx + ii), xi, px[k + 2]);
        ok &= to_primitive(u + 4 * ((int64_t)jj * nx + i), xi, py[k + 2]);
    }
    double fxp[4], fxm[4], fyp[4], fym[4];
    ok = ok && face_flux(px[1], px[2], px[3], px[4], 0, xi, eps, fxp) &&
         face_flux(px[0], px[1], px[2], px[3], 0, xi, eps, fxm) &&
         face_flux(py[1], py[2], py[3], py[4], 1, xi, eps, fyp) &&
         face_flux(py[0], py[1], py[2], py[3], 1, xi, eps, fym);
    if (!ok) {
        atomicMin(bad, (unsigned long long)c);
        return;
    }
    for (int k = 0; k < 4; ++k) out[4 * c + k] = -(fxp[k] - fxm[k]) / dx - (fyp[k] - fym[k]) / dy;
}

// u1 = u + dt l1  |  u = 0.5 u + 0.5 u1 + (0.5 dt) l2   (src/euler.cpp:175-180)
__global__ void rk2_combine_kernel(int stage, int64_t n, double dt, double* __restrict__ u, double* __restrict__ u1,
                                   const double* __restrict__ l) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    if (stage == 0) u1[k] = u[k] + dt * l[k];
    else u[k] = 0.5 * u[k] + 0.5 * u1[k] + (0.5 * dt) * l[k];
}

// moments_from_conserved (src/coupling.cpp:7-13): mom5 = (rho, ux, uy, 0, T)
__global__ void conserved_to_moments_kernel(const double* __restrict__ u, int64_t ncells, double hr,
                                            double* __restrict__ mom, unsigned long long* __restrict__ bad) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncells) return;
    const double* uc = u + 4 * c;
    double* m = mom + 5 * c;
    if (!(uc[0] > 0.0)) { atomicMin(bad, (unsigned long long)c); m[0] = 0.0; return; }
    const double p = (hr - 1.0) * (uc[3] - 0.5 * (uc[1] * uc[1] + uc[2] * uc[2]) / uc[0]);
    if (!(p > 0.0)) { atomicMin(bad, (unsigned long long)c); m[0] = 0.0; return; }
    m[0] = uc[0];
    m[1] = uc[1] / uc[0];
    m[2] = uc[2] / uc[0];
    m[3] = 0.0;
    m[4] = p / uc[0];
}

// conserved_from_moments (src/coupling.cpp:15-22)
__global__ void moments_to_conserved_kernel(const double* __restrict__ mom, int64_t ncells, double hr,
                                            double* __restrict__ u) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncells) return;
    const double* m = mom + 5 * c;
    const double rho = m[0];
    u[4 * c + 0] = rho;
    u[4 * c + 1] = rho * m[1];
    u[4 * c + 2] = rho * m[2];
    const double u2 = m[1] * m[1] + m[2] * m[2] + m[3] * m[3];
    u[4 * c + 3] = rho * m[4] / (hr - 1.0) + 0.5 * rho * u2;
}

// dst[k] = src[idx[k]] (gather, dir 0) or dst[idx[k]] = src[k] (scatter, dir 1), nb doubles per cell.
// One 256-thread CTA per cell block (grid-strided over the list), 8 16-byte loads in flight per thread.
__global__ void __launch_bounds__(256) cells_copy_kernel(int dir, int64_t nb, const int64_t* __restrict__ idx,
                                                         int64_t count, const double* __restrict__ src,
                                                         double* __restrict__ dst) {
    const int64_t n2 = nb / 2;
    for (int64_t k = blockIdx.x; k < count; k += gridDim.x) {
        const int64_t s = dir == 0 ? idx[k] : k, d = dir == 0 ? k : idx[k];
        const double2* sp = reinterpret_cast<const double2*>(src + s * nb);
        double2* dp = reinterpret_cast<double2*>(dst + d * nb);
        int64_t e = threadIdx.x;
        for (; e + 7 * 256 < n2; e += 8 * 256) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcs(sp + e + u * 256);
#pragma unroll
            for (int u = 0; u < 8; ++u) __stcs(dp + e + u * 256, v[u]);
        }
        for (; e < n2; e += 256) __stcs(dp + e, __ldcs(sp + e));
    }
}

unsigned long long* bad_slot(hk_ctx ctx) {
    if (!ctx->bad_flag) cudaMalloc(&ctx->bad_flag, sizeof(unsigned long long));
    return static_cast<unsigned long long*>(ctx->bad_flag);
}

int read_bad(hk_ctx ctx, unsigned long long* bad, const char* what) {
    unsigned long long h = ~0ull;
    int st = check_cuda(ctx, cudaMemcpyAsync(&h, bad, sizeof h, cudaMemcpyDeviceToHost, ctx->stream), what);
    if (!st) st = check_cuda(ctx, cudaStreamSynchronize(ctx->stream), what);
    if (st) return st;
    if (h != ~0ull) return fail(ctx, HK_POSITIVITY, std::string(what) + ": non-positive density or pressure", (int64_t)h);
    return HK_OK;
}

unsigned blocks(int64_t n, int t) { return unsigned((n + t - 1) / t); }

}  // namespace
}  // namespace hk

using namespace hk;

extern "C" {

int hk_euler_rhs_periodic(hk_ctx ctx, const double* u_dev, int nx, int ny, double dx, double dy, double xi,
                          double eps_weno, double* out_dev) {
    if (nx < 1 || ny < 1) return fail(ctx, HK_CONTRACT, "euler: empty grid");
    cudaSetDevice(ctx->device);
    unsigned long long* bad = bad_slot(ctx);
    cudaMemsetAsync(bad, 0xff, sizeof *bad, ctx->stream);
    euler_rhs_kernel<<<blocks((int64_t)nx * ny, 128), 128, 0, ctx->stream>>>(u_dev, nx, ny, dx, dy, xi, eps_weno, out_dev, bad);
    ctx->launches++;
    int st = check_cuda(ctx, cudaGetLastError(), "euler rhs");
    return st ? st : read_bad(ctx, bad, "euler_rhs_periodic");
}

int hk_euler_tvd_rk2_step(hk_ctx ctx, double* u_dev, int nx, int ny, double dx, double dy, double dt, double xi,
                          double eps_weno, double* work_dev) {
    HK_RANGE("hk_euler_tvd_rk2_step");
    if (nx < 1 || ny < 1) return fail(ctx, HK_CONTRACT, "euler: empty grid");
    cudaSetDevice(ctx->device);
    const int64_t n4 = 4LL * nx * ny;
    double* w = work_dev;
    if (!w) {  // the context's step workspace (kept across calls: no per-step allocation)
        const size_t need = sizeof(double) * 2 * n4;
        if (need > ctx->step_bytes) {
            if (ctx->step_work) {
                cudaStreamSynchronize(ctx->stream);
                cudaFree(ctx->step_work);
                ctx->step_work = nullptr;
                ctx->step_bytes = 0;
            }
            if (cudaMalloc(&ctx->step_work, need) != cudaSuccess) return fail(ctx, HK_CUDA, "euler step work alloc");
            ctx->step_bytes = need;
        }
        w = static_cast<double*>(ctx->step_work);
    }
    double *l = w, *u1 = w + n4;
    unsigned long long* bad = bad_slot(ctx);
    cudaMemsetAsync(bad, 0xff, sizeof *bad, ctx->stream);
    const unsigned gc = blocks((int64_t)nx * ny, 128), g4 = blocks(n4, 256);
    euler_rhs_kernel<<<gc, 128, 0, ctx->stream>>>(u_dev, nx, ny, dx, dy, xi, eps_weno, l, bad);
    rk2_combine_kernel<<<g4, 256, 0, ctx->stream>>>(0, n4, dt, u_dev, u1, l);
    euler_rhs_kernel<<<gc, 128, 0, ctx->stream>>>(u1, nx, ny, dx, dy, xi, eps_weno, l, bad);
    ctx->launches += 3;
    int st = check_cuda(ctx, cudaGetLastError(), "euler step");
    if (!st) st = read_bad(ctx, bad, "tvd_rk2_step_periodic");  // the reference throws before updating u
    if (!st) {
        rk2_combine_kernel<<<g4, 256, 0, ctx->stream>>>(1, n4, dt, u_dev, u1, l);
        ctx->launches++;
        st = check_cuda(ctx, cudaGetLastError(), "euler step");
    }
    return st;
}

int hk_conserved_to_maxwellian(hk_ctx ctx, int n, double vmax, const double* u_dev, int64_t ncells, double heat_ratio,
                               double* f_dev) {
    if (ncells <= 0) return HK_OK;
    cudaSetDevice(ctx->device);
    double* mom = nullptr;
    if (cudaMallocAsync(&mom, sizeof(double) * 5 * ncells, ctx->stream) != cudaSuccess)
        return fail(ctx, HK_CUDA, "transition alloc");
    unsigned long long* bad = bad_slot(ctx);
    cudaMemsetAsync(bad, 0xff, sizeof *bad, ctx->stream);
    conserved_to_moments_kernel<<<blocks(ncells, 128), 128, 0, ctx->stream>>>(u_dev, ncells, heat_ratio, mom, bad);
    ctx->launches++;
    int st = read_bad(ctx, bad, "moments_from_conserved");
    if (!st) st = maxwellian_launch(ctx, n, vmax, mom, ncells, f_dev, nullptr);
    cudaFreeAsync(mom, ctx->stream);
    return st;
}

int hk_distribution_to_conserved(hk_ctx ctx, int n, double vmax, const double* f_dev, int64_t ncells,
                                 double heat_ratio, double* u_dev) {
    if (ncells <= 0) return HK_OK;
    cudaSetDevice(ctx->device);
    double* mom = nullptr;
    int* status = nullptr;
    if (cudaMallocAsync(&mom, sizeof(double) * 5 * ncells, ctx->stream) != cudaSuccess ||
        cudaMallocAsync(&status, sizeof(int) * ncells, ctx->stream) != cudaSuccess)
        return fail(ctx, HK_CUDA, "transition alloc");
    int st = moments_launch(ctx, n, vmax, f_dev, ncells, mom, nullptr, nullptr, nullptr, status);
    if (!st) {
        moments_to_conserved_kernel<<<blocks(ncells, 128), 128, 0, ctx->stream>>>(mom, ncells, heat_ratio, u_dev);
        ctx->launches++;
        st = check_cuda(ctx, cudaGetLastError(), "moments_to_conserved");
    }
    if (!st) {  // moments_of throws degenerate_state_error on rho <= 0 or T <= 0
        std::vector<int> h(ncells);
        st = check_cuda(ctx, cudaMemcpyAsync(h.data(), status, sizeof(int) * ncells, cudaMemcpyDeviceToHost, ctx->stream),
                        "status");
        if (!st) st = check_cuda(ctx, cudaStreamSynchronize(ctx->stream), "status");
        for (int64_t c = 0; !st && c < ncells; ++c)
            if (h[c]) st = fail(ctx, h[c], "moments_of: degenerate state", c);
    }
    cudaFreeAsync(mom, ctx->stream);
    cudaFreeAsync(status, ctx->stream);
    return st;
}

int hk_gather_cells(hk_ctx ctx, int64_t nb, const double* src_dev, const int64_t* idx_dev, int64_t count, double* dst_dev) {
    if (count <= 0) return HK_OK;
    if (nb % 2) return fail(ctx, HK_CONTRACT, "gather: cell size must be even");
    cudaSetDevice(ctx->device);
    const unsigned grid = unsigned(std::min<int64_t>(count, int64_t(ctx->sm_count) * 8));
    cells_copy_kernel<<<grid, 256, 0, ctx->stream>>>(0, nb, idx_dev, count, src_dev, dst_dev);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "gather");
}

int hk_scatter_cells(hk_ctx ctx, int64_t nb, const double* src_dev, const int64_t* idx_dev, int64_t count, double* dst_dev) {
    if (count <= 0) return HK_OK;
    if (nb % 2) return fail(ctx, HK_CONTRACT, "scatter: cell size must be even");
    cudaSetDevice(ctx->device);
    const unsigned grid = unsigned(std::min<int64_t>(count, int64_t(ctx->sm_count) * 8));
    cells_copy_kernel<<<grid, 256, 0, ctx->stream>>>(1, nb, idx_dev, count, src_dev, dst_dev);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "scatter");
}

}  // extern "C"
