// hk_field.cu — spatial-field kernels: regime classifier (Algorithm 1) and the
// CWENO3 upwind kinetic transport sweep, sm_100a.
//
//   spatial_derivatives   src/indicators.cpp:14-32
//   v_eps1_eigenvalues    src/indicators.cpp:34-73
//   lambda_b_indicator    src/indicators.cpp:75-87
//   regime_update         src/regime.cpp:13-52
//   prim_from_moments     src/coupling.cpp:33-35
//   kinetic_transport_rhs src/transport.cpp:12-66, cweno3 src/euler.cpp:10-40
#include <cmath>
#include <cstdlib>

#include "hk_cells.cuh"
#include "hk_common.cuh"

namespace hk {

namespace {

// One thread per cell; periodic 4-neighbour stencil of prim = (rho, ux, uy, T).
__global__ void classify_kernel(ClassifyParams p, const double* __restrict__ mom, const double* __restrict__ eps_cell,
                                const double* __restrict__ l1, const int8_t* __restrict__ r_in,
                                int8_t* __restrict__ r_out, double* __restrict__ ind, int* __restrict__ status) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t cells = (int64_t)p.nx * p.ny;
    if (c >= cells) return;
    const int i = c % p.nx, j = c / p.nx;
    auto prim = [&](int ii, int jj, double (&q)[4]) {
        ii = (ii % p.nx + p.nx) % p.nx;
        jj = (jj % p.ny + p.ny) % p.ny;
        const double* m = mom + ((int64_t)jj * p.nx + ii) * 5;
        q[0] = m[0]; q[1] = m[1]; q[2] = m[2]; q[3] = m[4];  // prim_from_moments drops u_z
    };
    double pc[4], xm[4], xp[4], ym[4], yp[4];
    prim(i, j, pc); prim(i - 1, j, xm); prim(i + 1, j, xp); prim(i, j - 1, ym); prim(i, j + 1, yp);
    const double dx = p.dx, dy = p.dy;
    const double d_rho_x = (xp[0] - xm[0]) / (2.0 * dx);
    (void)d_rho_x;
    const double dux_dx = (xp[1] - xm[1]) / (2.0 * dx), dux_dy = (yp[1] - ym[1]) / (2.0 * dy);
    const double duy_dx = (xp[2] - xm[2]) / (2.0 * dx), duy_dy = (yp[2] - ym[2]) / (2.0 * dy);
    const double dT_dx = (xp[3] - xm[3]) / (2.0 * dx), dT_dy = (yp[3] - ym[3]) / (2.0 * dy);
    const double inv_dxdy = 1.0 / (dx * dy);
    const double lap_rho = (xm[0] + xp[0] + ym[0] + yp[0] - 4.0 * pc[0]) * inv_dxdy;
    const double lap_ux = (xm[1] + xp[1] + ym[1] + yp[1] - 4.0 * pc[1]) * inv_dxdy;
    const double lap_uy = (xm[2] + xp[2] + ym[2] + yp[2] - 4.0 * pc[2]) * inv_dxdy;
    const double eps = eps_cell[c];
    // v_eps1_coefficients / eigenvalues
    const double a1 = (4.0 / 3.0) * dux_dx - (2.0 / 3.0) * duy_dy;
    const double a2 = dT_dx * dT_dx;
    const double b1 = dux_dy + duy_dx;
    const double b2 = dT_dx * dT_dy;
    const double c1 = (4.0 / 3.0) * duy_dy - (2.0 / 3.0) * dux_dx;
    const double c2 = dT_dy * dT_dy;
    const double h1 = -(2.0 / 3.0) * (dux_dx + duy_dy);
    const double rho = pc[0], T = pc[3];
    const double mu = p.mu0 * sqrt(T), kappa = p.kappa0 * sqrt(T);
    const double xi1 = eps * mu / (rho * T);
    const double xi2 = eps * eps * 2.0 * kappa * kappa / (3.0 * rho * rho * T * T * T);
    const double gap = xi1 * (a1 - c1) + xi2 * (a2 - c2);
    const double dd = xi1 * b1 + xi2 * b2;
    const double root = sqrt(gap * gap + 4.0 * dd * dd);
    const double tr = -a1 * xi1 - a2 * xi2 - c1 * xi1 - c2 * xi2 + 2.0;
    const double la = 0.5 * (root + tr), lb = 0.5 * (-root + tr), lc = 1.0 - xi1 * h1;
    // lambda_B
    const double grad_t2 = dT_dx * dT_dx + dT_dy * dT_dy;
    const double grad_u2 = dux_dx * dux_dx + dux_dy * dux_dy + duy_dx * duy_dx + duy_dy * duy_dy;
    const double lap_u2 = p.signed_sum ? (lap_ux + lap_uy) * (lap_ux + lap_uy) : lap_ux * lap_ux + lap_uy * lap_uy;
    const double lrr = lap_rho / rho;
    const double lamB = eps * eps * (grad_t2 / T + grad_u2 + sqrt((lap_u2 + lrr * lrr) * (1.0 + T * T)));
    if (ind) {
        ind[c * 4 + 0] = la; ind[c * 4 + 1] = lb; ind[c * 4 + 2] = lc; ind[c * 4 + 3] = lamB;
    }
    // regime_update (src/regime.cpp:25-52); every indicator is available here
    const int r = r_in[c];
    const bool near = fabs(la - 1.0) <= p.eta0 && fabs(lb - 1.0) <= p.eta0 && fabs(lc - 1.0) <= p.eta0;
    int out = r, st = HK_OK;
    if (r == 2) out = fabs(lamB) > p.eta1 ? 2 : 1;
    else if (r == 1) {
        if (fabs(lamB) > p.eta1) out = 2;
        else if (near) {
            if (!l1) st = HK_CONTRACT;
            else out = l1[c] <= p.delta0 ? 0 : 1;
        } else out = 1;
    } else if (r == 0) out = near ? 0 : 1;
    else st = HK_CONTRACT;
    r_out[c] = (int8_t)out;
    if (status) status[c] = st;
}

__device__ __forceinline__ void cweno3(double um, double uc, double up, double eps, double& left, double& right) {
    const double sl = uc - um, sr = up - uc;
    const double b = 0.5 * (up - um);
    const double c = up - 2.0 * uc + um;
    const double is_l = sl * sl, is_r = sr * sr;
    const double is_c = (13.0 / 3.0) * c * c + b * b;
    double al = 0.25 / ((eps + is_l) * (eps + is_l));
    double ac = 0.50 / ((eps + is_c) * (eps + is_c));
    double ar = 0.25 / ((eps + is_r) * (eps + is_r));
    const double inv = 1.0 / (al + ac + ar);
    al *= inv; ac *= inv; ar *= inv;
    const double pc_a = uc - c / 12.0;
    const double c0 = al * uc + ar * uc + ac * pc_a;
    const double c1 = al * sl + ar * sr + ac * b;
    const double c2 = ac * c;
    left = c0 - 0.5 * c1 + 0.25 * c2;
    right = c0 + 0.5 * c1 + 0.25 * c2;
}

__device__ __forceinline__ double upwind_flux_diff(double v, const double (&s)[5], double eps) {
    double l, rp, rm;
    if (v > 0.0) {
        cweno3(s[1], s[2], s[3], eps, l, rp);
        cweno3(s[0], s[1], s[2], eps, l, rm);
        return v * (rp - rm);
    }
    double lp, lm, r;
    cweno3(s[2], s[3], s[4], eps, lp, r);
    cweno3(s[1], s[2], s[3], eps, lm, r);
    return v * (lp - lm);
}

// One thread per (cell, velocity node): 5-cell CWENO3 stencils in x and y.
// x_halo == -2: columns -2,-1 come from `lh` [ny][2][nb], nx,nx+1 from `rh`.
__global__ void __launch_bounds__(256) transport_kernel(TransportParams p, const double* __restrict__ f,
                                                        double* __restrict__ out, const double* __restrict__ lh,
                                                        const double* __restrict__ rh) {
    const int n = p.n;
    const int64_t nb = (int64_t)n * n * n;
    const int64_t total = (int64_t)p.nx * p.ny * nb;
    const int xh = p.x_halo > 0 ? p.x_halo : 0;
    const int nxi = p.nx + 2 * xh;  // input row length (cells)
    const double dv = 2.0 * p.vmax / n;
    const double inv_dx = 1.0 / p.dx, inv_dy = 1.0 / p.dy;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t idx = t % nb;
        const int64_t c = t / nb;
        const int i = c % p.nx, j = c / p.nx;
        const int k1 = idx / ((int64_t)n * n), k2 = (idx / n) % n;
        const double vx = -p.vmax + (k1 + 0.5) * dv, vy = -p.vmax + (k2 + 0.5) * dv;
        double sx[5], sy[5];
#pragma unroll
        for (int q = -2; q <= 2; ++q) {
            int ii = i + q;
            const int jj = ((j + q) % p.ny + p.ny) % p.ny;
            if (p.x_halo < 0 && ii < 0)
                sx[q + 2] = lh[((int64_t)j * p.lnx + (p.lnx + ii)) * nb + idx];
            else if (p.x_halo < 0 && ii >= p.nx)
                sx[q + 2] = rh[((int64_t)j * p.rnx + (ii - p.nx)) * nb + idx];
            else {
                if (p.x_halo == 0) ii = (ii % p.nx + p.nx) % p.nx;
                else ii += xh;
                sx[q + 2] = f[((int64_t)j * nxi + ii) * nb + idx];
            }
            sy[q + 2] = f[((int64_t)jj * nxi + i + xh) * nb + idx];
        }
        out[t] = -upwind_flux_diff(vx, sx, p.eps_weno) * inv_dx - upwind_flux_diff(vy, sy, p.eps_weno) * inv_dy;
    }
}

__global__ void axpby_kernel(int64_t count, double* __restrict__ out, const double* __restrict__ x, double a,
                             const double* __restrict__ y, double b, const double* __restrict__ z) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        double v = x[i];
        if (y) v += a * y[i];
        if (z) v += b * z[i];
        out[i] = v;
    }
}

}  // namespace

int classify_launch(hk_ctx ctx, const ClassifyParams& p, const double* mom, const double* eps_cell, const double* l1,
                    const int8_t* r_in, int8_t* r_out, double* ind, int* status) {
    const int64_t cells = (int64_t)p.nx * p.ny;
    if (cells <= 0) return HK_OK;
    classify_kernel<<<unsigned((cells + 127) / 128), 128, 0, ctx->stream>>>(p, mom, eps_cell, l1, r_in, r_out, ind,
                                                                           status);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "classify kernel");
}

bool transport_lanes_path(const TransportParams& p) {
    const int64_t nb = (int64_t)p.n * p.n * p.n;
    return (p.n & (p.n - 1)) == 0 && nb % 32 == 0 && p.ny >= 3;
}

int transport_launch(hk_ctx ctx, const TransportParams& p, const double* f, double* out, const double* lh,
                     const double* rh) {
    if ((p.out_pos || p.in_pos) && !transport_lanes_path(p))
        return fail(ctx, HK_CONTRACT, "transport: batch input / output needs the lane-per-column sweep");
    if (p.in_pos && (p.x_halo != 0 || !p.in_batch))
        return fail(ctx, HK_CONTRACT, "transport: batch input needs a periodic field and the batch");
    if (p.x_halo == 1 || p.x_halo < -2 || p.x_halo == -1 || (p.x_halo == -2 && (!lh || !rh)))
        return fail(ctx, HK_CONTRACT, "transport: x_halo must be 0, -2 (separate halo buffers) or >= 2");
    const int64_t total = (int64_t)p.nx * p.ny * p.n * p.n * p.n;
    if (total <= 0) return HK_OK;
    const int64_t nb = (int64_t)p.n * p.n * p.n;
    if (transport_lanes_path(p)) {  // lane-per-column sweep (hk_transport.cu)
        int lg = 0;
        while ((1 << lg) < p.n) ++lg;
        return transport_march_launch(ctx, p, lg, f, out, lh, rh);
    }
    const int64_t blocks = (total + 255) / 256;
    const int64_t cap = int64_t(ctx->sm_count) * 16;
    transport_kernel<<<unsigned(blocks < cap ? blocks : cap), 256, 0, ctx->stream>>>(p, f, out, lh, rh);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "transport kernel");
}

int axpby_launch(hk_ctx ctx, int64_t count, double* out, const double* x, double a, const double* y, double b,
                 const double* z) {
    if (count <= 0) return HK_OK;
    const int64_t blocks = (count + 255) / 256, cap = int64_t(ctx->sm_count) * 16;
    axpby_kernel<<<unsigned(blocks < cap ? blocks : cap), 256, 0, ctx->stream>>>(count, out, x, a, y, b, z);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "axpby kernel");
}

}  // namespace hk
