// hk_cells.cu — per-cell moment / relaxation / classification kernels, sm_100a.
//
// One 256-thread CTA per cell (grid-strided over the batch); the cell's N^3
// block is streamed from HBM with coalesced loads, reduced in registers +
// warp shuffles, and the few scalar solves (3x3 Cholesky test, 5x5 complete-
// pivoting LU) run on one thread.  These paths are HBM-bound (16 N^3 bytes
// per cell-step); every pass after the first re-reads the block from L2.
//
// Reference functions (src/ = /root/reference/proj/core/src):
//   moments_of             src/moments.cpp:21-53
//   second_moment          src/moments.cpp:55-81
//   maxwellian             src/moments.cpp:88-112
//   anisotropic_gaussian   src/moments.cpp:120-157
//   match_moments          src/moments.cpp:164-246
//   remove_invariant_moments src/moments.cpp:192-267
//   realizability_matrix   src/moments.cpp:269-312
//   l1_distance_to_maxwellian src/indicators.cpp:89-98
//   penalized_residual     src/boltzmann.cpp:9-27   (after the collision kernel)
//   penalized_stage_solve  src/boltzmann.cpp:29-45
//   esbgk_stage_solve      src/esbgk.cpp:9-45
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "hk_cells.cuh"
#include "hk_common.cuh"
#include "hk_internal.h"

namespace hk {

namespace {

constexpr int NT = 256;

struct VGrid {
    int n;
    double vmax, dv, dvk;
    __device__ double node(int k) const { return -vmax + (k + 0.5) * dv; }
};

__host__ VGrid make_vgrid(int n, double vmax) {
    VGrid g;
    g.n = n;
    g.vmax = vmax;
    g.dv = 2.0 * vmax / n;
    g.dvk = g.dv * g.dv * g.dv;
    return g;
}

// Block-wide sum of K doubles; result valid in every thread.
template <int K>
__device__ void block_sum(double (&v)[K], double* scratch /* [8][K] */) {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) scratch[w * K + k] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double s = 0.0;
#pragma unroll
        for (int ww = 0; ww < NT / 32; ++ww) s += scratch[ww * K + k];
        v[k] = s;
    }
}

// Eigen::FullPivLU<Matrix<double,5,5>> (src/moments.cpp:215-221), as
// oracle/hk_oracle.c:hko_solve5.  Returns false when singular.
// Register-resident form: every index is a compile-time constant after
// unrolling; the data-dependent pivot row / column swaps are selects (no
// local memory).  Same pivot order (first maximum in column-major scan) as the
// scalar algorithm; the multipliers use one reciprocal of the pivot per step
// (a_ik * (1 / a_kk): within an ulp of the division, a shorter latency chain).
__device__ __forceinline__ bool solve5(const double a_in[25], const double rhs[5], double x[5]) {
    double a[5][5];
    int rp[5], cp[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
#pragma unroll
        for (int j = 0; j < 5; ++j) a[i][j] = a_in[5 * i + j];
        rp[i] = cp[i] = i;
    }
    double maxpivot = 0.0;
    int nonzero = 5;
    bool live = true;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        int bi = k, bj = k;
        double big = -1.0;
#pragma unroll
        for (int j = k; j < 5; ++j)
#pragma unroll
            for (int i = k; i < 5; ++i) {
                const double v = fabs(a[i][j]);
                const bool gt = v > big;
                big = gt ? v : big;
                bi = gt ? i : bi;
                bj = gt ? j : bj;
            }
        if (live && big == 0.0) {
            nonzero = k;
            live = false;
        }
        if (live) {
            if (big > maxpivot) maxpivot = big;
#pragma unroll
            for (int r = k + 1; r < 5; ++r) {  // rows k <-> bi
                const bool sw = bi == r;
#pragma unroll
                for (int j = 0; j < 5; ++j) {
                    const double t = a[k][j];
                    a[k][j] = sw ? a[r][j] : t;
                    a[r][j] = sw ? t : a[r][j];
                }
                const int ti = rp[k];
                rp[k] = sw ? rp[r] : ti;
                rp[r] = sw ? ti : rp[r];
            }
#pragma unroll
            for (int c = k + 1; c < 5; ++c) {  // columns k <-> bj
                const bool sw = bj == c;
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    const double t = a[i][k];
                    a[i][k] = sw ? a[i][c] : t;
                    a[i][c] = sw ? t : a[i][c];
                }
                const int ti = cp[k];
                cp[k] = sw ? cp[c] : ti;
                cp[c] = sw ? ti : cp[c];
            }
            const double rkk = 1.0 / a[k][k];  // one division per step (the multipliers: l_ik = a_ik / a_kk)
#pragma unroll
            for (int i = k + 1; i < 5; ++i) {
                a[i][k] *= rkk;
#pragma unroll
                for (int j = k + 1; j < 5; ++j) a[i][j] -= a[i][k] * a[k][j];
            }
        }
    }
    const double thr = 2.220446049250313e-16 * 5.0 * maxpivot;
    int rank = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) rank += (i < nonzero && fabs(a[i][i]) > thr) ? 1 : 0;
    if (rank != 5) return false;
    double y[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        double v = rhs[0];
#pragma unroll
        for (int r = 1; r < 5; ++r) v = rp[i] == r ? rhs[r] : v;
        y[i] = v;
    }
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int j = 0; j < i; ++j) y[i] -= a[i][j] * y[j];
    double rd[5];  // the diagonal's reciprocals, independent of each other: off the back-substitution chain
#pragma unroll
    for (int i = 0; i < 5; ++i) rd[i] = 1.0 / a[i][i];
#pragma unroll
    for (int i = 4; i >= 0; --i) {
#pragma unroll
        for (int j = i + 1; j < 5; ++j) y[i] -= a[i][j] * y[j];
        y[i] *= rd[i];
    }
#pragma unroll
    for (int o = 0; o < 5; ++o) {
        double v = 0.0;
#pragma unroll
        for (int i = 0; i < 5; ++i) v = cp[i] == o ? y[i] : v;
        x[o] = v;
    }
    return true;
}

struct Mom {
    double rho, ux, uy, uz, T;
};

// Pass 1 sums (k3-inner partials not reproduced; order differs by round-off):
// s0, sx, sy, sz, s2, and the raw second moment xx, xy, xz, yy, yz, zz.
__device__ void raw_sums(const double* __restrict__ f, const VGrid& g, double (&s)[11], double* scratch) {
    const int n = g.n;
    const int nb = n * n * n;
#pragma unroll
    for (int k = 0; k < 11; ++k) s[k] = 0.0;
    for (int idx = threadIdx.x; idx < nb; idx += NT) {
        const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
        const double vx = g.node(k1), vy = g.node(k2), vz = g.node(k3);
        const double w = f[idx];
        s[0] += w;
        s[1] += vx * w;
        s[2] += vy * w;
        s[3] += vz * w;
        s[4] += (vx * vx + vy * vy + vz * vz) * w;
        s[5] += vx * vx * w;
        s[6] += vx * vy * w;
        s[7] += vx * vz * w;
        s[8] += vy * vy * w;
        s[9] += vy * vz * w;
        s[10] += vz * vz * w;
    }
    block_sum<11>(s, scratch);
}

// moments_of (src/moments.cpp:44-52).  Returns HK_DEGENERATE on rho<=0 / T<=0.
__device__ int moments_from_sums(const double (&s)[11], const VGrid& g, Mom& m) {
    m.rho = s[0] * g.dvk;
    m.ux = s[1] / s[0];
    m.uy = s[2] / s[0];
    m.uz = s[3] / s[0];
    m.T = (s[4] / s[0] - (m.ux * m.ux + m.uy * m.uy + m.uz * m.uz)) / 3.0;
    if (!(m.rho > 0.0)) return HK_DEGENERATE;
    if (!(m.T > 0.0)) return HK_DEGENERATE;
    return HK_OK;
}

__device__ double energy_of(const Mom& m) {
    return 0.5 * m.rho * (m.ux * m.ux + m.uy * m.uy + m.uz * m.uz) + 1.5 * m.rho * m.T;
}

// Separable Maxwellian factors ex/ey/ez in shared memory (src/moments.cpp:93-102).
__device__ double maxwell_factors(const Mom& m, const VGrid& g, double* ex, double* ey, double* ez) {
    const double inv2T = 0.5 / m.T;
    for (int k = threadIdx.x; k < g.n; k += NT) {
        const double v = g.node(k);
        ex[k] = exp(-(v - m.ux) * (v - m.ux) * inv2T);
        ey[k] = exp(-(v - m.uy) * (v - m.uy) * inv2T);
        ez[k] = exp(-(v - m.uz) * (v - m.uz) * inv2T);
    }
    __syncthreads();
    return m.rho / pow(2.0 * M_PI * m.T, 1.5);
}

// Coupling matrix A_rc = sum phi_r psi_c w dvK of a weight given node-wise by
// `wfun(idx, vx, vy, vz)` (src/moments.cpp:164-189).
template <typename WF>
__device__ void coupling(const VGrid& g, const double uc[3], WF wfun, double (&A)[25], double* scratch) {
    const int n = g.n, nb = n * n * n;
#pragma unroll
    for (int i = 0; i < 25; ++i) A[i] = 0.0;
    for (int idx = threadIdx.x; idx < nb; idx += NT) {
        const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
        const double vx = g.node(k1), vy = g.node(k2), vz = g.node(k3);
        const double w = wfun(idx, vx, vy, vz);
        const double cx = vx - uc[0], cy = vy - uc[1], cz = vz - uc[2];
        const double c2 = cx * cx + cy * cy + cz * cz;
        const double v2 = vx * vx + vy * vy + vz * vz;
        const double psi[5] = {1.0, cx, cy, cz, c2};
        const double phi[5] = {1.0, vx, vy, vz, v2};
#pragma unroll
        for (int r = 0; r < 5; ++r)
#pragma unroll
            for (int c = 0; c < 5; ++c) A[5 * r + c] += phi[r] * psi[c] * w;
    }
    block_sum<25>(A, scratch);
#pragma unroll
    for (int i = 0; i < 25; ++i) A[i] *= g.dvk;
}

__device__ __forceinline__ double quad_factor(const double x[5], double vx, double vy, double vz, const double uc[3]) {
    const double cx = vx - uc[0], cy = vy - uc[1], cz = vz - uc[2];
    const double c2 = cx * cx + cy * cy + cz * cz;
    return x[0] + x[1] * cx + x[2] * cy + x[3] * cz + x[4] * c2;
}

// ---------------------------------------------------------------------------
// moments + second moment + realizability + L1 distance, one CTA per cell
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) moments_kernel(const double* __restrict__ f, int64_t ncells, VGrid g,
                                                     double* __restrict__ mom, double* __restrict__ sigma,
                                                     double* __restrict__ real, double* __restrict__ l1,
                                                     int* __restrict__ status, const int64_t* __restrict__ src_idx,
                                                     const int* __restrict__ count_dev) {
    __shared__ double scratch[8 * 25];
    __shared__ double ex[128], ey[128], ez[128];
    const int n = g.n, nb = n * n * n;
    if (count_dev) ncells = min(ncells, (int64_t)*count_dev);
    for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
        const double* fc = f + (src_idx ? src_idx[cell] : cell) * nb;
        double s[11];
        raw_sums(fc, g, s, scratch);
        Mom m;
        const int st = moments_from_sums(s, g, m);
        if (threadIdx.x == 0) {
            if (mom) {
                double* o = mom + cell * 5;
                o[0] = m.rho; o[1] = m.ux; o[2] = m.uy; o[3] = m.uz; o[4] = m.T;
            }
            if (sigma) {
                double* o = sigma + cell * 6;
                for (int k = 0; k < 6; ++k) o[k] = s[5 + k] * g.dvk;  // xx xy xz yy yz zz
            }
            if (status) status[cell] = st;
        }
        if (st != HK_OK || (!real && !l1)) continue;
        // pass 2: realizability (src/moments.cpp:269-312) and L1 distance
        const double pref = l1 ? maxwell_factors(m, g, ex, ey, ez) : 0.0;
        const double ist = 1.0 / sqrt(m.T);
        double r[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) r[k] = 0.0;
        for (int idx = threadIdx.x; idx < nb; idx += NT) {
            const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
            const double Vx = (g.node(k1) - m.ux) * ist, Vy = (g.node(k2) - m.uy) * ist, Vz = (g.node(k3) - m.uz) * ist;
            const double w = fc[idx];
            const double V2 = Vx * Vx + Vy * Vy + Vz * Vz;
            r[0] += Vx * Vx * w;
            r[1] += Vx * Vy * w;
            r[2] += Vx * Vz * w;
            r[3] += Vy * Vy * w;
            r[4] += Vy * Vz * w;
            r[5] += Vz * Vz * w;
            const double bw = 0.5 * (V2 - 5.0) * w;
            r[6] += bw * Vx;
            r[7] += bw * Vy;
            r[8] += bw * Vz;
            const double e = 0.5 * V2 - 2.5;
            r[9] += e * e * w;
            if (l1) r[10] += fabs(w - pref * ex[k1] * ey[k2] * ez[k3]);
        }
        block_sum<11>(r, scratch);
        if (threadIdx.x == 0) {
            if (real) {
                const double sc = g.dvk / m.rho;
                double s2[6];
                for (int k = 0; k < 6; ++k) s2[k] = r[k] * sc;
                const double tr3 = (s2[0] + s2[3] + s2[5]) / 3.0;
                double* o = real + cell * 13;  // a_bar (3x3 row-major), b_bar, c_bar
                o[0] = s2[0] - tr3; o[1] = s2[1]; o[2] = s2[2];
                o[3] = s2[1]; o[4] = s2[3] - tr3; o[5] = s2[4];
                o[6] = s2[2]; o[7] = s2[4]; o[8] = s2[5] - tr3;
                o[9] = r[6] * sc; o[10] = r[7] * sc; o[11] = r[8] * sc;
                o[12] = 0.4 * r[9] * sc;
            }
            if (l1) l1[cell] = r[10] * g.dvk;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Maxwellian of given moments (src/moments.cpp:88-112)
// ---------------------------------------------------------------------------
// dst_idx (optional): cell k is written to block dst_idx[k]; count_dev
// (optional): the list length lives on the device (at most ncells).
__global__ void __launch_bounds__(NT) maxwellian_kernel(const double* __restrict__ mom, int64_t ncells, VGrid g,
                                                        double* __restrict__ out, int* __restrict__ status,
                                                        const int64_t* __restrict__ dst_idx,
                                                        const int* __restrict__ count_dev) {
    __shared__ double ex[128], ey[128], ez[128];
    const int n = g.n, nb = n * n * n;
    if (count_dev) ncells = min(ncells, (int64_t)*count_dev);
    for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
        Mom m{mom[cell * 5], mom[cell * 5 + 1], mom[cell * 5 + 2], mom[cell * 5 + 3], mom[cell * 5 + 4]};
        const bool ok = (m.rho > 0.0) && (m.T > 0.0);
        if (threadIdx.x == 0 && status) status[cell] = ok ? HK_OK : HK_DEGENERATE;
        if (!ok) continue;
        const double pref = maxwell_factors(m, g, ex, ey, ez);
        double* o = out + (dst_idx ? dst_idx[cell] : cell) * nb;
        for (int idx = threadIdx.x; idx < nb; idx += NT) {
            const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
            o[idx] = pref * ex[k1] * ey[k2] * ez[k3];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Relaxation stages: f = (eps f* + A G~)/(eps + A), G~ the moment-matched
// Maxwellian (penalized, src/boltzmann.cpp:29-45) or anisotropic Gaussian
// (ES-BGK, src/esbgk.cpp:9-45).  Three passes: sums of f*, coupling matrix
// of G (G recomputed, never stored), blend.
// info[cell] = status | (gaussian_fallback << 8)
// ---------------------------------------------------------------------------
template <bool ESBGK>
__global__ void __launch_bounds__(NT) stage_kernel(const double* __restrict__ fin, double* __restrict__ out,
                                                   int64_t ncells, VGrid g, double a, const double* __restrict__ eps_cell,
                                                   double eps_scalar, double beta, double coeff,
                                                   int* __restrict__ info, double* __restrict__ mom_out) {
    __shared__ double scratch[8 * 25];
    __shared__ double ex[128], ey[128], ez[128];
    __shared__ double par[16];  // [0..8] inverse Tc, [9] pref, [10] use_gauss, [11..15] x
    const int n = g.n, nb = n * n * n;
    for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
        const double* fc = fin + cell * nb;
        double* oc = out + cell * nb;
        const double eps = eps_cell ? eps_cell[cell] : eps_scalar;
        double s[11];
        raw_sums(fc, g, s, scratch);
        Mom m;
        int st = moments_from_sums(s, g, m);
        if (threadIdx.x == 0 && mom_out) {
            double* o = mom_out + cell * 5;
            o[0] = m.rho; o[1] = m.ux; o[2] = m.uy; o[3] = m.uz; o[4] = m.T;
        }
        const double A = ESBGK ? a * (coeff * m.rho) : a * (coeff * m.rho);  // nu = coeff rho | beta = coeff rho
        if (st != HK_OK || !(A > 0.0)) {
            if (threadIdx.x == 0 && info) info[cell] = st;
            if (st == HK_OK)
                for (int idx = threadIdx.x; idx < nb; idx += NT) oc[idx] = fc[idx];  // identity stage
            __syncthreads();
            continue;
        }
        int fallback = 0;
        if (ESBGK && threadIdx.x == 0) {
            // Sigma blend toward rho (T I + u u^T) (src/esbgk.cpp:24-33)
            const double omb = 1.0 - beta;
            const double u[3] = {m.ux, m.uy, m.uz};
            const int map[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
            double theta[9], tc[9];
            const double denom = eps + omb * A, oa = omb * A;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    const double sstar = s[5 + map[3 * i + j]] * g.dvk;
                    const double siso = m.rho * ((i == j ? m.T : 0.0) + u[i] * u[j]);
                    const double sstage = (eps * sstar + oa * siso) / denom;
                    theta[3 * i + j] = sstage / m.rho - u[i] * u[j];
                }
            const double iso = (1.0 - beta) * m.T;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) tc[3 * i + j] = (i == j ? iso : 0.0) + beta * theta[3 * i + j];
            // Eigen::LLT info (src/moments.cpp:128-134)
            double l[9] = {0};
            bool ok = true;
            for (int k = 0; k < 3 && ok; ++k) {
                double x = tc[3 * k + k];
                for (int j = 0; j < k; ++j) x -= l[3 * k + j] * l[3 * k + j];
                if (!(x > 0.0)) { ok = false; break; }
                l[3 * k + k] = sqrt(x);
                for (int i = k + 1; i < 3; ++i) {
                    double y = tc[3 * i + k];
                    for (int j = 0; j < k; ++j) y -= l[3 * i + j] * l[3 * k + j];
                    l[3 * i + k] = y / l[3 * k + k];
                }
            }
            if (ok) {
                const double* q = tc;
                const double c00 = q[4] * q[8] - q[5] * q[7], c01 = q[5] * q[6] - q[3] * q[8], c02 = q[3] * q[7] - q[4] * q[6];
                const double det = q[0] * (q[4] * q[8] - q[5] * q[7]) - q[1] * (q[3] * q[8] - q[5] * q[6]) +
                                   q[2] * (q[3] * q[7] - q[4] * q[6]);
                const double dinv = q[0] * c00 + q[1] * c01 + q[2] * c02;
                const double id = 1.0 / dinv;
                par[0] = c00 * id; par[1] = (q[2] * q[7] - q[1] * q[8]) * id; par[2] = (q[1] * q[5] - q[2] * q[4]) * id;
                par[3] = c01 * id; par[4] = (q[0] * q[8] - q[2] * q[6]) * id; par[5] = (q[2] * q[3] - q[0] * q[5]) * id;
                par[6] = c02 * id; par[7] = (q[1] * q[6] - q[0] * q[7]) * id; par[8] = (q[0] * q[4] - q[1] * q[3]) * id;
                par[9] = m.rho / sqrt(pow(2.0 * M_PI, 3) * det);
                par[10] = 1.0;
            } else {
                par[10] = 0.0;  // fall back to the Maxwellian
            }
        }
        __syncthreads();
        const bool gauss = ESBGK && par[10] != 0.0;
        if (ESBGK) fallback = gauss ? 0 : 1;
        double pref = 0.0;
        if (!gauss) pref = maxwell_factors(m, g, ex, ey, ez);
        // equilibrium value at node idx, recomputed in passes 2 and 3
        auto eq = [&](int idx, double vx, double vy, double vz) -> double {
            const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
            if (!gauss) return pref * ex[k1] * ey[k2] * ez[k3];
            const double dx = vx - m.ux, dy = vy - m.uy, dz = vz - m.uz;
            const double qxy = par[0] * dx * dx + 2.0 * par[1] * dx * dy + par[4] * dy * dy;
            const double lz = 2.0 * (par[2] * dx + par[5] * dy);
            const double q = qxy + dz * (lz + par[8] * dz);
            return par[9] * exp(-0.5 * q);
        };
        // match_moments(G, rho, rho u, E) (src/moments.cpp:225-246)
        const double mom3[3] = {m.rho * m.ux, m.rho * m.uy, m.rho * m.uz};
        const double uc[3] = {mom3[0] / m.rho, mom3[1] / m.rho, mom3[2] / m.rho};
        double Amat[25];
        coupling(g, uc, eq, Amat, scratch);
        if (threadIdx.x == 0) {
            const double rhs[5] = {m.rho, mom3[0], mom3[1], mom3[2], 2.0 * energy_of(m)};
            double x[5];
            const bool ok = solve5(Amat, rhs, x);
            for (int k = 0; k < 5; ++k) par[11 + k] = x[k];
            st = ok ? HK_OK : HK_DEGENERATE;
            if (info) info[cell] = st | (fallback << 8);
            scratch[0] = st;
        }
        __syncthreads();
        st = (int)scratch[0];
        if (st == HK_OK) {
            const double x[5] = {par[11], par[12], par[13], par[14], par[15]};
            const double wf = eps / (eps + A), wg = A / (eps + A);
            for (int idx = threadIdx.x; idx < nb; idx += NT) {
                const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
                const double vx = g.node(k1), vy = g.node(k2), vz = g.node(k3);
                const double G = eq(idx, vx, vy, vz) * quad_factor(x, vx, vy, vz, uc);
                oc[idx] = wf * fc[idx] + wg * G;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// penalized_residual epilogue (src/boltzmann.cpp:14-26): q holds Q(f) on
// entry and Q(f) + beta (f - M~) with the invariant moments removed on exit.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) residual_finish_kernel(const double* __restrict__ f, double* __restrict__ q,
                                                             int64_t ncells, VGrid g, double pen_coeff,
                                                             int* __restrict__ status) {
    __shared__ double scratch[8 * 25];
    __shared__ double ex[128], ey[128], ez[128];
    __shared__ double par[12];
    const int n = g.n, nb = n * n * n;
    for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
        const double* fc = f + cell * nb;
        double* qc = q + cell * nb;
        double s[11];
        raw_sums(fc, g, s, scratch);
        Mom m;
        int st = moments_from_sums(s, g, m);
        if (st != HK_OK) {
            if (threadIdx.x == 0 && status) status[cell] = st;
            __syncthreads();
            continue;
        }
        const double beta = pen_coeff * m.rho;
        const double pref = maxwell_factors(m, g, ex, ey, ez);
        const double mom3[3] = {m.rho * m.ux, m.rho * m.uy, m.rho * m.uz};
        const double uc[3] = {mom3[0] / m.rho, mom3[1] / m.rho, mom3[2] / m.rho};
        auto maxw = [&](int idx, double, double, double) -> double {
            const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
            return pref * ex[k1] * ey[k2] * ez[k3];
        };
        double Amat[25];
        coupling(g, uc, maxw, Amat, scratch);
        if (threadIdx.x == 0) {
            const double rhs[5] = {m.rho, mom3[0], mom3[1], mom3[2], 2.0 * energy_of(m)};
            double x[5];
            const bool ok = solve5(Amat, rhs, x);
            for (int k = 0; k < 5; ++k) par[k] = x[k];
            scratch[0] = ok ? HK_OK : HK_DEGENERATE;
        }
        __syncthreads();
        st = (int)scratch[0];
        __syncthreads();
        if (st != HK_OK) {
            if (threadIdx.x == 0 && status) status[cell] = st;
            continue;
        }
        const double x[5] = {par[0], par[1], par[2], par[3], par[4]};
        // out = Q + beta (f - M~); then remove_invariant_moments(out, M~, u)
        // (src/moments.cpp:248-267) with uc = u.
        const double u3[3] = {m.ux, m.uy, m.uz};
        auto mt = [&](int idx, double vx, double vy, double vz) -> double {
            return maxw(idx, vx, vy, vz) * quad_factor(x, vx, vy, vz, uc);
        };
        double B[25];
        coupling(g, u3, mt, B, scratch);
        double inv[5] = {0, 0, 0, 0, 0};
        for (int idx = threadIdx.x; idx < nb; idx += NT) {
            const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
            const double vx = g.node(k1), vy = g.node(k2), vz = g.node(k3);
            const double o = qc[idx] + beta * (fc[idx] - mt(idx, vx, vy, vz));
            qc[idx] = o;
            inv[0] += o;
            inv[1] += vx * o;
            inv[2] += vy * o;
            inv[3] += vz * o;
            inv[4] += (vx * vx + vy * vy + vz * vz) * o;
        }
        block_sum<5>(inv, scratch);
        if (threadIdx.x == 0) {
            double rhs[5], y[5];
            for (int k = 0; k < 5; ++k) rhs[k] = inv[k] * g.dvk;
            const bool ok = solve5(B, rhs, y);
            for (int k = 0; k < 5; ++k) par[5 + k] = y[k];
            if (status) status[cell] = ok ? HK_OK : HK_DEGENERATE;
            scratch[0] = ok ? HK_OK : HK_DEGENERATE;
        }
        __syncthreads();
        if ((int)scratch[0] == HK_OK) {
            const double y[5] = {par[5], par[6], par[7], par[8], par[9]};
            for (int idx = threadIdx.x; idx < nb; idx += NT) {
                const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
                const double vx = g.node(k1), vy = g.node(k2), vz = g.node(k3);
                qc[idx] -= quad_factor(y, vx, vy, vz, u3) * mt(idx, vx, vy, vz);
            }
        }
        __syncthreads();
    }
}

// ===========================================================================
// Streaming CTA-per-cell kernels (n a power of two, 8 <= n <= 64; the
// production path): 256 threads stream a cell's block as double2 pairs with
// many loads in flight, two CTAs per SM; the kernels above (thread-per-cell
// loops) serve every other n.  (Warp-per-cell variants were measured slower
// at n >= 8 and removed; they spilled.)
// ===========================================================================

template <int K>
__device__ __forceinline__ void warp_sum(double (&v)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
}

__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

// L2 eviction-priority hints (createpolicy): a cell's block read in a first
// pass and again in a last pass is loaded evict_last, its final reads and the
// outputs evict_first, so the re-read finds it in L2.
#ifndef HK_STAGE_HINTS
#define HK_STAGE_HINTS 1
#endif
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ldg2_hint(const double* ptr, uint64_t pol) {
#if HK_STAGE_HINTS
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n" : "=d"(v.x), "=d"(v.y) : "l"(ptr), "l"(pol));
    return v;
#else
    (void)pol;
    return ldg2(ptr);
#endif
}
__device__ __forceinline__ void st2_hint(double* ptr, double2 v, uint64_t pol) {
#if HK_STAGE_HINTS
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(ptr), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
#else
    (void)pol;
    *reinterpret_cast<double2*>(ptr) = v;
#endif
}

// Coupling matrix from the 14 weighted monomial moments of w (degree <= 4)
// instead of 25 direct products: A = sum phi psi^T w with psi affine in
// (1, v, |v|^2) (src/moments.cpp:164-189 evaluates the same sums directly).
__device__ void coupling_from_monomials(const double (&M)[14], const double uc[3], double dvk, double (&A)[25]);

// A_rc = sum phi_r psi_c w dvK from the 14 weighted monomial moments of w.
__device__ void coupling_from_monomials(const double (&M)[14], const double uc[3], double dvk, double (&A)[25]) {
    const double M0 = M[0];
    const double M1[3] = {M[1], M[2], M[3]};
    const double M2[3][3] = {{M[4], M[5], M[6]}, {M[5], M[7], M[8]}, {M[6], M[8], M[9]}};
    const double M3[3] = {M[10], M[11], M[12]};
    const double M4 = M[13];
    const double Mv2 = M2[0][0] + M2[1][1] + M2[2][2];
    const double U2 = uc[0] * uc[0] + uc[1] * uc[1] + uc[2] * uc[2];
    const double ucM1 = uc[0] * M1[0] + uc[1] * M1[1] + uc[2] * M1[2];
    const double ucM3 = uc[0] * M3[0] + uc[1] * M3[1] + uc[2] * M3[2];
    A[0] = M0;
    for (int i = 0; i < 3; ++i) A[1 + i] = M1[i] - uc[i] * M0;
    A[4] = Mv2 - 2.0 * ucM1 + U2 * M0;
    for (int j = 0; j < 3; ++j) {
        A[5 * (1 + j)] = M1[j];
        for (int i = 0; i < 3; ++i) A[5 * (1 + j) + 1 + i] = M2[j][i] - uc[i] * M1[j];
        const double ucM2j = uc[0] * M2[j][0] + uc[1] * M2[j][1] + uc[2] * M2[j][2];
        A[5 * (1 + j) + 4] = M3[j] - 2.0 * ucM2j + U2 * M1[j];
    }
    A[20] = Mv2;
    for (int i = 0; i < 3; ++i) A[21 + i] = M3[i] - uc[i] * Mv2;
    A[24] = M4 - 2.0 * ucM3 + U2 * Mv2;
#pragma unroll
    for (int i = 0; i < 25; ++i) A[i] *= dvk;
}




// ---------------------------------------------------------------------------
// moments + second moment + realizability + L1, one 512-thread CTA per cell,
// one CTA per SM (grid = SM count): the 148 blocks in flight (37 MB at N = 32)
// stay in L2, so the L1 pass re-reads the block from L2, not HBM.
// Realizability from ONE pass of raw monomial moments up to degree 4
// (S, S_i, S_ij, R_i = sum |v|^2 v_i f, Q4 = sum |v|^4 f) via the central-
// moment identities (c = v - u):
//   C_ij          = S_ij - u_i u_j S
//   sum |c|^2 c_i = R_i - u_i P - 2 (S2 u)_i + 2 u_i |u|^2 S,   P = tr S2
//   sum |c|^4     = Q4 + 4 u.S2.u - 4 u.R + 2 |u|^2 P - 3 |u|^4 S
// (src/moments.cpp:269-312 sums the same quantities over V = c / sqrt(T)
// directly; the identities are exact, cancellation costs ~|u|^4 / T^2 ulps).
// ---------------------------------------------------------------------------
#ifndef HK_MOM_UNROLL
#define HK_MOM_UNROLL 8  // loads in flight per thread: 2 -> 7.4 ms, 4 -> 6.0, 8 -> 5.8 (config 3)
#endif
constexpr int kMomUnroll = HK_MOM_UNROLL;
template <int MT, int MINB, int UNR = kMomUnroll>
__global__ void __launch_bounds__(MT, MINB) moments_cta_kernel(const double* __restrict__ f, int64_t ncells, VGrid g,
                                                            int lg, double* __restrict__ mom, double* __restrict__ sigma,
                                                            double* __restrict__ real, double* __restrict__ l1,
                                                            int* __restrict__ status, const int64_t* __restrict__ src_idx,
                                                     const int* __restrict__ count_dev) {
    __shared__ double red[MT / 32][16];
    __shared__ double tabs[3][128];
    __shared__ double2 xpow[128][2];  // (vx, vx^2), (vx^3, vx^4) per k1
    __shared__ double bc[8];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = g.n, nb = n * n * n;
    if (count_dev) ncells = min(ncells, (int64_t)*count_dev);
    for (int k = t; k < n; k += MT) {
        const double v = g.node(k), v2 = v * v;
        xpow[k][0] = make_double2(v, v2);
        xpow[k][1] = make_double2(v2 * v, v2 * v2);
    }
    __syncthreads();
    const uint64_t pol_last = l2_evict_last(), pol_first = l2_evict_first();
    for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
        const double* fc = f + (src_idx ? src_idx[cell] : cell) * nb;
        double M[14];  // S, Sx, Sy, Sz, Sxx, Sxy, Sxz, Syy, Syz, Szz, Rx, Ry, Rz, Q4
#pragma unroll
        for (int k = 0; k < 14; ++k) M[k] = 0.0;
        // Column form: a thread owns the k1-columns of two adjacent (k2, k3)
        // nodes and accumulates A_a = sum_k1 vx^a f (a <= 4: 5 fp64 per node,
        // vx powers from shared memory); the 14 moments follow per column from
        // A_a and the column's (vy, vz) (src/moments.cpp:21-86 sums the same
        // monomials; only the summation order differs).
        for (int cp = t; cp < (n << lg) / 2; cp += MT) {
            const int col = 2 * cp, k2 = col >> lg, k3 = col & (n - 1);
            const double* fcol = fc + col;
            double A0[5] = {0, 0, 0, 0, 0}, A1[5] = {0, 0, 0, 0, 0};
#pragma unroll UNR
            for (int k1 = 0; k1 < n; ++k1) {
                const double2 w = ldg2_hint(fcol + ((int64_t)k1 << (2 * lg)), l1 ? pol_last : pol_first);
                const double2 p12 = xpow[k1][0], p34 = xpow[k1][1];
                A0[0] += w.x; A1[0] += w.y;
                A0[1] += p12.x * w.x; A1[1] += p12.x * w.y;
                A0[2] += p12.y * w.x; A1[2] += p12.y * w.y;
                A0[3] += p34.x * w.x; A1[3] += p34.x * w.y;
                A0[4] += p34.y * w.x; A1[4] += p34.y * w.y;
            }
            const double vy = g.node(k2), yy = vy * vy;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double* A = h ? A1 : A0;
                const double vz = g.node(k3 + h), rho2 = yy + vz * vz;
                M[0] += A[0];
                M[1] += A[1];
                M[2] += vy * A[0];
                M[3] += vz * A[0];
                M[4] += A[2];
                M[5] += vy * A[1];
                M[6] += vz * A[1];
                M[7] += yy * A[0];
                M[8] += vy * (vz * A[0]);
                M[9] += vz * (vz * A[0]);
                const double b = A[2] + rho2 * A[0];
                M[10] += A[3] + rho2 * A[1];
                M[11] += vy * b;
                M[12] += vz * b;
                M[13] += A[4] + rho2 * (2.0 * A[2] + rho2 * A[0]);
            }
        }
#pragma unroll
        for (int k = 0; k < 14; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) M[k] += __shfl_xor_sync(0xffffffffu, M[k], o);
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < 14; ++k) red[warp][k] = M[k];
        __syncthreads();
        if (t == 0) {
            double S[14];
            for (int k = 0; k < 14; ++k) {
                double v = 0.0;
                for (int w2 = 0; w2 < MT / 32; ++w2) v += red[w2][k];
                S[k] = v;
            }
            const double s11[11] = {S[0], S[1], S[2], S[3], S[4] + S[7] + S[9], S[4], S[5], S[6], S[7], S[8], S[9]};
            Mom m;
            const int st = moments_from_sums(s11, g, m);
            if (mom) {
                double* o = mom + cell * 5;
                o[0] = m.rho; o[1] = m.ux; o[2] = m.uy; o[3] = m.uz; o[4] = m.T;
            }
            if (sigma)
                for (int k = 0; k < 6; ++k) sigma[cell * 6 + k] = s11[5 + k] * g.dvk;
            if (status) status[cell] = st;
            if (st == HK_OK && real) {
                const double u[3] = {m.ux, m.uy, m.uz};
                const double S2[3][3] = {{S[4], S[5], S[6]}, {S[5], S[7], S[8]}, {S[6], S[8], S[9]}};
                const double R[3] = {S[10], S[11], S[12]};
                const double S0 = S[0], P = S[4] + S[7] + S[9];
                const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
                double C[3][3], c3[3], S2u[3];
                for (int i = 0; i < 3; ++i) {
                    S2u[i] = S2[i][0] * u[0] + S2[i][1] * u[1] + S2[i][2] * u[2];
                    for (int j = 0; j < 3; ++j) C[i][j] = S2[i][j] - u[i] * u[j] * S0;
                    c3[i] = R[i] - u[i] * P - 2.0 * S2u[i] + 2.0 * u[i] * uu * S0;
                }
                const double uS2u = u[0] * S2u[0] + u[1] * S2u[1] + u[2] * S2u[2];
                const double uR = u[0] * R[0] + u[1] * R[1] + u[2] * R[2];
                const double c4 = S[13] + 4.0 * uS2u - 4.0 * uR + 2.0 * uu * P - 3.0 * uu * uu * S0;
                const double c2 = C[0][0] + C[1][1] + C[2][2];
                const double T = m.T, iS = 1.0 / S0;
                double s2[3][3];
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) s2[i][j] = C[i][j] / T * iS;
                const double tr3 = (s2[0][0] + s2[1][1] + s2[2][2]) / 3.0;
                double* o = real + cell * 13;
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 3; ++j) o[3 * i + j] = s2[i][j] - (i == j ? tr3 : 0.0);
                const double it32 = 1.0 / (T * sqrt(T));
                for (int i = 0; i < 3; ++i) o[9 + i] = 0.5 * c3[i] * it32 * iS;  // sum (|V|^2 - 5)/2 V_i f / S
                // C = 0.4 sum (|V|^2/2 - 5/2)^2 f / S = 0.4 (|V|^4/4 - 5/2 |V|^2 + 25/4) averaged
                o[12] = 0.4 * (0.25 * c4 / (T * T) - 2.5 * c2 / T + 6.25 * S0) * iS;
            }
            bc[0] = st;
            bc[1] = m.rho; bc[2] = m.ux; bc[3] = m.uy; bc[4] = m.uz; bc[5] = m.T;
        }
        __syncthreads();
        if (l1 && bc[0] == 0.0) {
            Mom m{bc[1], bc[2], bc[3], bc[4], bc[5]};
            const double inv2T = 0.5 / m.T;
            for (int k = t; k < n; k += MT) {
                const double v = g.node(k);
                tabs[0][k] = exp(-(v - m.ux) * (v - m.ux) * inv2T);
                tabs[1][k] = exp(-(v - m.uy) * (v - m.uy) * inv2T);
                tabs[2][k] = exp(-(v - m.uz) * (v - m.uz) * inv2T);
            }
            const double pref = m.rho / pow(2.0 * M_PI * m.T, 1.5);
            __syncthreads();
            double acc = 0.0;
            for (int cp = t; cp < (n << lg) / 2; cp += MT) {  // same column form
                const int col = 2 * cp, k2 = col >> lg, k3 = col & (n - 1);
                const double* fcol = fc + col;
                const double py0 = pref * tabs[1][k2] * tabs[2][k3], py1 = pref * tabs[1][k2] * tabs[2][k3 + 1];
#pragma unroll UNR
                for (int k1 = 0; k1 < n; ++k1) {
                    const double2 w = ldg2_hint(fcol + ((int64_t)k1 << (2 * lg)), pol_first);
                    const double ex = tabs[0][k1];
                    acc += fabs(w.x - py0 * ex) + fabs(w.y - py1 * ex);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) red[warp][15] = acc;
            __syncthreads();
            if (t == 0) {
                double v = 0.0;
                for (int w2 = 0; w2 < MT / 32; ++w2) v += red[w2][15];
                l1[cell] = v * g.dvk;
            }
        }
        __syncthreads();  // red / tabs / bc reused by the next cell
    }
}

// ---------------------------------------------------------------------------
// penalized_residual epilogue (src/boltzmann.cpp:14-26), one CTA per cell,
// TWO streaming passes: q holds Q(f) on entry and
//   Q + beta (f - M~) - (y0 + y.d + y4 |d|^2) M~
// on exit.  The moment-matching and invariant-removal coupling matrices
// (src/moments.cpp:164-189) are sums of polynomials times the Maxwellian M,
// which is separable along (vx, vy, vz) in shifted coordinates, so both are
// assembled from 1-D sums  C_a = sum_k (v_k - uc)^a e(k),  D_a = sum_k (v_k - u)^a e(k)
// (a <= 4 / 6, e the per-axis Maxwellian factors) instead of two passes over
// the N^3 nodes; the invariant moments of Q + beta (f - M~) follow from pass-1
// sums of q and f and the closed-form moments of M~ (same quantities as the
// reference's node sums, different rounding).  Pass 1 reads f and q in column
// form (5 sums each), pass 2 reads both again and writes q.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 ld2_hint(const double* ptr, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n" : "=d"(v.x), "=d"(v.y) : "l"(ptr), "l"(pol));
    return v;
}

// sum of coef_i coef_j X[a_i + a_j] Y[b_i + b_j] Z[c_i + c_j] over two term lists
struct PolyT {
    double c;
    int a, b, z;
};
__device__ double poly_pair_sum(const PolyT* p, int np, const PolyT* q, int nq, const double* X, const double* Y,
                                const double* Z) {
    double acc = 0.0;
    for (int i = 0; i < np; ++i)
        for (int j = 0; j < nq; ++j)
            acc += p[i].c * q[j].c * X[p[i].a + q[j].a] * Y[p[i].b + q[j].b] * Z[p[i].z + q[j].z];
    return acc;
}
// phi = (1, v, |v|^2) written in coordinates w = v - s (shift s): lists of terms
__device__ int phi_terms(int r, const double s[3], PolyT* o) {
    if (r == 0) { o[0] = {1.0, 0, 0, 0}; return 1; }
    if (r <= 3) {
        o[0] = {1.0, r == 1, r == 2, r == 3};
        o[1] = {s[r - 1], 0, 0, 0};
        return 2;
    }
    o[0] = {1.0, 2, 0, 0}; o[1] = {1.0, 0, 2, 0}; o[2] = {1.0, 0, 0, 2};
    o[3] = {2.0 * s[0], 1, 0, 0}; o[4] = {2.0 * s[1], 0, 1, 0}; o[5] = {2.0 * s[2], 0, 0, 1};
    o[6] = {s[0] * s[0] + s[1] * s[1] + s[2] * s[2], 0, 0, 0};
    return 7;
}
// psi = (1, w, |w|^2) in the same coordinates
__device__ int psi_terms(int c, PolyT* o) {
    if (c == 0) { o[0] = {1.0, 0, 0, 0}; return 1; }
    if (c <= 3) { o[0] = {1.0, c == 1, c == 2, c == 3}; return 1; }
    o[0] = {1.0, 2, 0, 0}; o[1] = {1.0, 0, 2, 0}; o[2] = {1.0, 0, 0, 2};
    return 3;
}

#ifndef HK_RES_MT
#define HK_RES_MT 256
#endif
#ifndef HK_RES_MINB
#define HK_RES_MINB 2
#endif
template <int MT, int MINB>
__global__ void __launch_bounds__(MT, MINB) residual_cta_kernel(const double* __restrict__ f, double* __restrict__ q,
                                                                int64_t ncells, VGrid g, int lg, double pen_coeff,
                                                                int* __restrict__ status) {
    __shared__ double red[MT / 32][10];
    __shared__ double tab[3][128];       // Maxwellian factors e_x, e_y, e_z
    __shared__ double sums[2][3][8];     // C_a (uc-centred, a <= 4) and D_a (u-centred, a <= 6) per axis
    __shared__ double par[24];           // [0] status, [1..5] m, [6] pref, [7..11] x, [12..16] y, [17] beta, [18..20] uc
    __shared__ double mat[32];           // coupling matrix entries / invariants, one per lane of warp 0
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int n = g.n, nb = n * n * n;
    const uint64_t pol_keep = l2_evict_last(), pol_last = l2_evict_first();
    for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
        const double* fc = f + cell * nb;
        double* qc = q + cell * nb;
        // ---- pass 1: (1, v, |v|^2) sums of f and of q, column form ----
        double S[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) S[k] = 0.0;
        for (int cp = t; cp < (n << lg) / 2; cp += MT) {
            const int col = 2 * cp, k2 = col >> lg, k3 = col & (n - 1);
            double A[2][2][3] = {};  // [f | q][node of the pair][sum_k1 vx^a w], a <= 2
#pragma unroll 4
            for (int k1 = 0; k1 < n; ++k1) {
                const int64_t o = ((int64_t)k1 << (2 * lg)) + col;
                const double2 wf = ldg2_hint(fc + o, pol_keep), wq = ld2_hint(qc + o, pol_keep);
                const double vx = g.node(k1), xx = vx * vx;
                A[0][0][0] += wf.x; A[0][0][1] += vx * wf.x; A[0][0][2] += xx * wf.x;
                A[0][1][0] += wf.y; A[0][1][1] += vx * wf.y; A[0][1][2] += xx * wf.y;
                A[1][0][0] += wq.x; A[1][0][1] += vx * wq.x; A[1][0][2] += xx * wq.x;
                A[1][1][0] += wq.y; A[1][1][1] += vx * wq.y; A[1][1][2] += xx * wq.y;
            }
            const double vy = g.node(k2);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double vz = g.node(k3 + h), r2 = vy * vy + vz * vz;
#pragma unroll
                for (int w = 0; w < 2; ++w) {
                    double* s = S + 5 * w;
                    s[0] += A[w][h][0];
                    s[1] += A[w][h][1];
                    s[2] += vy * A[w][h][0];
                    s[3] += vz * A[w][h][0];
                    s[4] += A[w][h][2] + r2 * A[w][h][0];
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 10; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) S[k] += __shfl_xor_sync(0xffffffffu, S[k], o);
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < 10; ++k) red[warp][k] = S[k];
        __syncthreads();
        if (t == 0) {
            for (int k = 0; k < 10; ++k) {
                double v = 0.0;
                for (int w2 = 0; w2 < MT / 32; ++w2) v += red[w2][k];
                S[k] = v;
            }
            Mom m;
            const double s11[11] = {S[0], S[1], S[2], S[3], S[4], 0, 0, 0, 0, 0, 0};
            const int st = moments_from_sums(s11, g, m);
            par[0] = st;
            par[1] = m.rho; par[2] = m.ux; par[3] = m.uy; par[4] = m.uz; par[5] = m.T;
            for (int k = 0; k < 10; ++k) red[0][k] = S[k];  // keep the block sums for thread 0's solves
        }
        __syncthreads();
        if (par[0] != 0.0) {
            if (t == 0 && status) status[cell] = (int)par[0];
            __syncthreads();
            continue;
        }
        const Mom m{par[1], par[2], par[3], par[4], par[5]};
        const double mom3[3] = {m.rho * m.ux, m.rho * m.uy, m.rho * m.uz};
        const double uc[3] = {mom3[0] / m.rho, mom3[1] / m.rho, mom3[2] / m.rho};  // match_moments' centre
        const double u3[3] = {m.ux, m.uy, m.uz};                                      // remove_invariant_moments' centre
        {   // Maxwellian factors (src/moments.cpp:93-102) and the 1-D shifted power sums
            const double inv2T = 0.5 / m.T;
            for (int k = t; k < n; k += MT) {
                const double v = g.node(k);
                tab[0][k] = exp(-(v - m.ux) * (v - m.ux) * inv2T);
                tab[1][k] = exp(-(v - m.uy) * (v - m.uy) * inv2T);
                tab[2][k] = exp(-(v - m.uz) * (v - m.uz) * inv2T);
            }
            __syncthreads();
            if (t < 6) {  // (set, axis): C (uc-centred) for t < 3, D (u-centred) for t >= 3
                const int set = t / 3, ax = t % 3;
                const double sh = set ? u3[ax] : uc[ax];
                double acc[7] = {0, 0, 0, 0, 0, 0, 0};
                for (int k = 0; k < n; ++k) {
                    const double w = g.node(k) - sh, e = tab[ax][k];
                    double p = e;
#pragma unroll
                    for (int a = 0; a < 7; ++a) {
                        acc[a] += p;
                        p *= w;
                    }
                }
                for (int a = 0; a < 7; ++a) sums[set][ax][a] = acc[a];
            }
            __syncthreads();
        }
        // ---- coupling matrices and solves: warp 0, one matrix entry per lane ----
        if (warp == 0) {
            const double pref = m.rho / pow(2.0 * M_PI * m.T, 1.5);  // maxwell_factors' prefactor
            const double sc = pref * g.dvk;
            PolyT pt[7], qt[3];
            // match_moments of M (src/moments.cpp:225-246): A_rc = sum phi_r psi_c M dvK, coordinates c = v - uc
            if (lane < 25) {
                const int r0 = lane / 5, c0 = lane % 5;
                const int np = phi_terms(r0, uc, pt), nq = psi_terms(c0, qt);
                mat[lane] = sc * poly_pair_sum(pt, np, qt, nq, sums[0][0], sums[0][1], sums[0][2]);
            }
            __syncwarp();
            if (lane == 0) {
                double A[25];
                for (int k = 0; k < 25; ++k) A[k] = mat[k];
                const double rhs[5] = {m.rho, mom3[0], mom3[1], mom3[2], 2.0 * energy_of(m)};
                double x[5] = {0, 0, 0, 0, 0};
                const bool ok = solve5(A, rhs, x);
                for (int k = 0; k < 5; ++k) par[7 + k] = x[k];
                par[0] = ok ? HK_OK : HK_DEGENERATE;
            }
            __syncwarp();
            // M~ = M (x0 + x.c + x4 |c|^2) written in d = v - u: c = d + delta, delta = u - uc
            const double x[5] = {par[7], par[8], par[9], par[10], par[11]};
            const double dl[3] = {u3[0] - uc[0], u3[1] - uc[1], u3[2] - uc[2]};
            const PolyT mt[7] = {{x[0] + x[1] * dl[0] + x[2] * dl[1] + x[3] * dl[2] +
                                      x[4] * (dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2]), 0, 0, 0},
                                 {x[1] + 2.0 * x[4] * dl[0], 1, 0, 0},
                                 {x[2] + 2.0 * x[4] * dl[1], 0, 1, 0},
                                 {x[3] + 2.0 * x[4] * dl[2], 0, 0, 1},
                                 {x[4], 2, 0, 0},
                                 {x[4], 0, 2, 0},
                                 {x[4], 0, 0, 2}};
            // remove_invariant_moments (src/moments.cpp:248-267) with weight M~, centre u:
            // B_rc = sum phi_r psi_c M~ dvK (coordinates d); lanes 25..29: the moments of M~
            const double beta = pen_coeff * m.rho;
            if (lane < 30) {
                const int r0 = lane < 25 ? lane / 5 : lane - 25;
                const int np = phi_terms(r0, u3, pt);
                PolyT pm[49];
                int npm = 0;
                for (int i2 = 0; i2 < np; ++i2)
                    for (int j2 = 0; j2 < 7; ++j2)
                        pm[npm++] = {pt[i2].c * mt[j2].c, pt[i2].a + mt[j2].a, pt[i2].b + mt[j2].b, pt[i2].z + mt[j2].z};
                if (lane < 25) {
                    const int nq = psi_terms(lane % 5, qt);
                    mat[lane] = sc * poly_pair_sum(pm, npm, qt, nq, sums[1][0], sums[1][1], sums[1][2]);
                } else {
                    const PolyT one = {1.0, 0, 0, 0};
                    const double mtil = sc * poly_pair_sum(pm, npm, &one, 1, sums[1][0], sums[1][1], sums[1][2]);
                    mat[lane] = (red[0][5 + r0] + beta * red[0][r0]) * g.dvk - beta * mtil;  // invariants of Q + beta (f - M~)
                }
            }
            __syncwarp();
            if (lane == 0) {
                double B[25], inv[5], y[5] = {0, 0, 0, 0, 0};
                for (int k = 0; k < 25; ++k) B[k] = mat[k];
                for (int k = 0; k < 5; ++k) inv[k] = mat[25 + k];
                bool ok = par[0] == HK_OK;
                if (ok) ok = solve5(B, inv, y);
                par[0] = ok ? HK_OK : HK_DEGENERATE;
                par[6] = pref;
                for (int k = 0; k < 5; ++k) par[12 + k] = y[k];
                par[17] = beta;
                if (status) status[cell] = ok ? HK_OK : HK_DEGENERATE;
            }
        }
        __syncthreads();
        if (par[0] == 0.0) {
            // ---- pass 2: q <- q + beta (f - M~) - (y0 + y.d + y4 |d|^2) M~ ----
            const double pref = par[6], beta = par[17];
            const double x0 = par[7], x1 = par[8], x2 = par[9], x3 = par[10], x4 = par[11];
            const double y0 = par[12], y1 = par[13], y2 = par[14], y3 = par[15], y4 = par[16];
            for (int cp = t; cp < (n << lg) / 2; cp += MT) {
                const int col = 2 * cp, k2 = col >> lg, k3 = col & (n - 1);
                const double vy = g.node(k2);
                const double cy = vy - uc[1], dy = vy - u3[1];
                double pz[2], cz[2], dz[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double vz = g.node(k3 + h);
                    cz[h] = vz - uc[2];
                    dz[h] = vz - u3[2];
                    pz[h] = pref * tab[1][k2] * tab[2][k3 + h];
                }
#pragma unroll 4
                for (int k1 = 0; k1 < n; ++k1) {
                    const int64_t o = ((int64_t)k1 << (2 * lg)) + col;
                    const double2 wf = ldg2_hint(fc + o, pol_last);
                    double2 wq = ld2_hint(qc + o, pol_last);
                    const double vx = g.node(k1), ex = tab[0][k1];
                    const double cx = vx - uc[0], dx = vx - u3[0];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const double Mv = pz[h] * ex;
                        const double mt = Mv * (x0 + x1 * cx + x2 * cy + x3 * cz[h] + x4 * (cx * cx + cy * cy + cz[h] * cz[h]));
                        const double corr = (y0 + y1 * dx + y2 * dy + y3 * dz[h] + y4 * (dx * dx + dy * dy + dz[h] * dz[h])) * mt;
                        const double fv = h ? wf.y : wf.x;
                        double& qv = h ? wq.y : wq.x;
                        qv = qv + beta * (fv - mt) - corr;
                    }
                    st2_hint(qc + o, wq, pol_last);
                }
            }
        }
        __syncthreads();  // red / tab / sums / par reused by the next cell
    }
}

// ---------------------------------------------------------------------------
// Stage solves (penalized / ES-BGK), one 256-thread CTA per cell, 3 CTAs per
// SM (the cells in flight stay in L2 between the first and last pass).  A
// thread owns groups of 4 consecutive k3 nodes of one (k1, k2) pencil.  The
// equilibrium is evaluated WITHOUT a per-node exp: for the Gaussian
//   exp(-1/2 d^T S d) = P(k1,k2) R(k1,k2)^k3 Z(k3),
//   P = pref exp(-Q12/2 - L dz0),  R = exp(-L dv),  Z = exp(-S33 dz^2 / 2),
//   L = S13 dx + S23 dy  (dz = dz0 + k3 dv on the uniform grid),
// with P, R per pencil and Z per k3 in shared memory (N^2 + N exps per cell
// instead of 2 N^3) and R^k3 by a branch-free square-and-multiply; cells whose
// exponent ranges could overflow take the direct exp.  The Maxwellian is the
// separable special case (R = 1).  Same passes as stage_kernel:
// raw sums -> Sigma / LLT / inverse -> coupling matrix (14 monomial moments of
// the equilibrium) -> FullPivLU solve -> blended output.
// ---------------------------------------------------------------------------
// 14 monomial moments (S, S_i, S_ij, R_i, Q4) of a pencil from its k3 sums m_c = sum z^c e
__device__ __forceinline__ void acc14(double (&M)[14], double vx, double vy, double m0, double m1, double m2, double m3,
                                      double m4) {
    const double xx = vx * vx, yy = vy * vy, r2 = xx + yy;
    M[0] += m0;
    M[1] += vx * m0; M[2] += vy * m0; M[3] += m1;
    M[4] += xx * m0; M[5] += vx * (vy * m0); M[6] += vx * m1;
    M[7] += yy * m0; M[8] += vy * m1; M[9] += m2;
    const double aa = r2 * m0 + m2;
    M[10] += vx * aa; M[11] += vy * aa; M[12] += r2 * m1 + m3;
    M[13] += r2 * (r2 * m0 + 2.0 * m2) + m4;
}

// Bank swizzle of the pass-3 (Z, ZQ) table: the 8 threads of a pencil read
// entries 4 s + j (s = 0..7) at once; slot = k ^ ((k >> 3) & 3) in the low
// three bits puts them in 8 distinct 16-byte bank groups.
__device__ __forceinline__ int zq_slot(int k) { return (k & ~7) | ((k & 7) ^ ((k >> 3) & 3)); }

#ifndef HK_STAGE_U1
#define HK_STAGE_U1 8  // pass-1 loads in flight: 2 -> 15.4 ms, 4 -> 14.7, 8 -> 14.3 (config 3 ES-BGK stage)
#endif
#ifndef HK_STAGE_U2
#define HK_STAGE_U2 1
#endif
#ifndef HK_STAGE_U3
#define HK_STAGE_U3 1
#endif
constexpr int kStageU1 = HK_STAGE_U1, kStageU2 = HK_STAGE_U2, kStageU3 = HK_STAGE_U3;
#ifndef HK_STAGE_PROF
#define HK_STAGE_PROF 0  // per-phase clocks of thread 0 (profiling builds)
#endif
#if HK_STAGE_PROF
__device__ unsigned long long g_stage_prof[5];
#endif
// Explicit accumulation fused into the stage input (ACC): the stage solves
// f* = f + cq q1 + ck k1 (the PR(2,2,2) f_acc of src/boltzmann.cpp:80-81 /
// src/esbgk.cpp:68-72), formed on the fly in passes 1 and 3 instead of a
// separate combination pass writing f_acc (one field write + read saved).
struct AccIn {
    const double* q1;
    const double* k1;
    double cq, ck;
};
template <bool ESBGK, int MT, int MINB, bool ACC = false>
__global__ void __launch_bounds__(MT, MINB) stage_cta_kernel(const double* __restrict__ fin, double* __restrict__ out,
                                                             int64_t ncells, VGrid g, int lg, double a,
                                                             const double* __restrict__ eps_cell, double eps_scalar,
                                                             double beta, double coeff, int* __restrict__ info,
                                                             double* __restrict__ mom_out, double* __restrict__ k1_out,
                                                             double k1_scale, AccIn acc) {
    extern __shared__ double dsm[];
    const int n = g.n, nb = n * n * n, ngroups = nb >> 2;
    double* Ptab = dsm;            // [n*n]
    double* Rtab = Ptab + n * n;   // [n*n]
    double* Ztab = Rtab + n * n;   // [n]
    double* red = Ztab + n;        // [MT/32][16]
    double* par = red + (MT / 32) * 16;  // [32]
    double2* xpow = reinterpret_cast<double2*>(par + 32);  // [n] (vx, vx^2)
    double* Htab = par + 32 + 2 * n;   // [n][6]: z^c Z(k3), c <= 4 (pass-2 Horner coefficients)
    double2* ZQ = reinterpret_cast<double2*>(Htab + 6 * n);  // [n]: (Z, Z Q) of pass 3
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    auto block_reduce = [&](double* v, int K) {  // sum of K values over the CTA -> par[16..16+K) (K <= 14)
        for (int k = 0; k < K; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if (lane == 0)
            for (int k = 0; k < K; ++k) red[warp * 16 + k] = v[k];
        __syncthreads();
        if (t < K) {
            double s = 0.0;
            for (int w2 = 0; w2 < MT / 32; ++w2) s += red[w2 * 16 + t];
            par[16 + t] = s;
        }
        __syncthreads();
    };
    for (int k = t; k < n; k += MT) {
        const double v = g.node(k);
        xpow[k] = make_double2(v, v * v);
    }
    __syncthreads();
    const uint64_t pol_last = l2_evict_last(), pol_first = l2_evict_first();
#if HK_STAGE_PROF
    long long sp[5] = {0, 0, 0, 0, 0}, st0 = clock64();
#define SP_MARK(k) do { if (t == 0) { const long long _c = clock64(); sp[k] += _c - st0; st0 = _c; } } while (0)
#else
#define SP_MARK(k) do {} while (0)
#endif
    for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
        const double* fc = fin + cell * nb;
        double* oc = out + cell * nb;
        const double eps = eps_cell ? eps_cell[cell] : eps_scalar;
        // ---- pass 1: raw sums, column form (moments_cta_kernel): a thread owns the
        // k1-columns of two adjacent (k2, k3) nodes, A_a = sum_k1 vx^a f (a <= 2) ----
        {
            double s[11];
#pragma unroll
            for (int k = 0; k < 11; ++k) s[k] = 0.0;
            for (int cp = t; cp < (n << lg) / 2; cp += MT) {
                const int col = 2 * cp, k2 = col >> lg, k3 = col & (n - 1);
                const double* fcol = fc + col;
                double A[2][3] = {{0, 0, 0}, {0, 0, 0}};
#pragma unroll (ACC ? 4 : kStageU1)
                for (int k1 = 0; k1 < n; ++k1) {
                    double2 w;
                    if constexpr (ACC) {  // f_acc formed here and parked in `out` for pass 3 (L2-resident)
                        const int64_t o = col + ((int64_t)k1 << (2 * lg));
                        const double2 fv = ldg2_hint(fcol + ((int64_t)k1 << (2 * lg)), pol_first);
                        const double2 qv = ldg2_hint(acc.q1 + cell * nb + o, pol_first);
                        const double2 kv = ldg2_hint(acc.k1 + cell * nb + o, pol_first);
                        w = make_double2(fv.x + acc.cq * qv.x + acc.ck * kv.x, fv.y + acc.cq * qv.y + acc.ck * kv.y);
                        st2_hint(oc + o, w, pol_last);
                    } else {
                        w = ldg2_hint(fcol + ((int64_t)k1 << (2 * lg)), pol_last);
                    }
                    const double2 p = xpow[k1];
                    A[0][0] += w.x; A[1][0] += w.y;
                    A[0][1] += p.x * w.x; A[1][1] += p.x * w.y;
                    A[0][2] += p.y * w.x; A[1][2] += p.y * w.y;
                }
                const double vy = g.node(k2);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double vz = g.node(k3 + h);
                    s[0] += A[h][0];
                    s[1] += A[h][1];
                    s[2] += vy * A[h][0];
                    s[3] += vz * A[h][0];
                    s[4] += A[h][2] + (vy * vy + vz * vz) * A[h][0];
                    s[5] += A[h][2];
                    s[6] += vy * A[h][1];
                    s[7] += vz * A[h][1];
                    s[8] += vy * (vy * A[h][0]);
                    s[9] += vy * (vz * A[h][0]);
                    s[10] += vz * (vz * A[h][0]);
                }
            }
            block_reduce(s, 11);
        }
        double s11[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) s11[k] = par[16 + k];
        Mom m;
        int st = moments_from_sums(s11, g, m);
        if (t == 0 && mom_out) {
            double* o = mom_out + cell * 5;
            o[0] = m.rho; o[1] = m.ux; o[2] = m.uy; o[3] = m.uz; o[4] = m.T;
        }
        const double A = a * (coeff * m.rho);  // a nu (nu = coeff rho) | a beta_pen (beta = coeff rho)
        if (st != HK_OK || !(A > 0.0)) {
            if (t == 0 && info) info[cell] = st;
            if (st == HK_OK && !ACC)  // identity stage (with ACC, pass 1 already left f_acc in out)
                for (int q = t; q < ngroups; q += MT) {
                    const int idx = 4 * q;
                    *reinterpret_cast<double2*>(oc + idx) = ldg2(fc + idx);
                    *reinterpret_cast<double2*>(oc + idx + 2) = ldg2(fc + idx + 2);
                    if (k1_out) {  // identity stage: k1 = 0
                        *reinterpret_cast<double2*>(k1_out + cell * nb + idx) = make_double2(0.0, 0.0);
                        *reinterpret_cast<double2*>(k1_out + cell * nb + idx + 2) = make_double2(0.0, 0.0);
                    }
                }
            __syncthreads();
            continue;
        }
        SP_MARK(0);
        // ---- ES-BGK tensor (src/esbgk.cpp:24-33) + LLT test + inverse, thread 0 ----
        if (t == 0) {
            par[0] = 0.0;  // use_gauss
            if (ESBGK) {
                const double omb = 1.0 - beta;
                const double u[3] = {m.ux, m.uy, m.uz};
                const int map[9] = {0, 1, 2, 1, 3, 4, 2, 4, 5};
                double tc[9];
                const double denom = eps + omb * A, oa = omb * A;
                const double iso = (1.0 - beta) * m.T;
                const double idr = 1.0 / (denom * m.rho);  // one division for the 9 entries
                // the 9 entries are independent: unrolled
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        const double sstar = s11[5 + map[3 * i + j]] * g.dvk;
                        const double siso = m.rho * ((i == j ? m.T : 0.0) + u[i] * u[j]);
                        const double theta = (eps * sstar + oa * siso) * idr - u[i] * u[j];
                        tc[3 * i + j] = (i == j ? iso : 0.0) + beta * theta;
                    }
                double l[9] = {0};
                bool ok = true;
                for (int k = 0; k < 3 && ok; ++k) {
                    double x = tc[3 * k + k];
                    for (int j = 0; j < k; ++j) x -= l[3 * k + j] * l[3 * k + j];
                    if (!(x > 0.0)) { ok = false; break; }
                    l[3 * k + k] = sqrt(x);
                    for (int i = k + 1; i < 3; ++i) {
                        double y = tc[3 * i + k];
                        for (int j = 0; j < k; ++j) y -= l[3 * i + j] * l[3 * k + j];
                        l[3 * i + k] = y / l[3 * k + k];
                    }
                }
                if (ok) {
                    const double* q = tc;
                    const double c00 = q[4] * q[8] - q[5] * q[7], c01 = q[5] * q[6] - q[3] * q[8], c02 = q[3] * q[7] - q[4] * q[6];
                    const double det = q[0] * (q[4] * q[8] - q[5] * q[7]) - q[1] * (q[3] * q[8] - q[5] * q[6]) +
                                       q[2] * (q[3] * q[7] - q[4] * q[6]);
                    const double id = 1.0 / (q[0] * c00 + q[1] * c01 + q[2] * c02);
                    par[1] = c00 * id; par[2] = (q[2] * q[7] - q[1] * q[8]) * id; par[3] = (q[1] * q[5] - q[2] * q[4]) * id;
                    par[4] = (q[0] * q[8] - q[2] * q[6]) * id; par[5] = (q[2] * q[3] - q[0] * q[5]) * id;
                    par[6] = (q[0] * q[4] - q[1] * q[3]) * id;  // S11 S12 S13 S22 S23 S33
                    par[7] = m.rho / sqrt(248.05021344239853 * det);  // (2 pi)^3
                    par[0] = 1.0;
                }
            }
            par[8] = 0.0;  // direct-exp flag (set below if a table factor could overflow)
        }
        __syncthreads();
        const bool gauss = par[0] != 0.0;
        const int fallback = (ESBGK && !gauss) ? 1 : 0;
        const double S11 = par[1], S12 = par[2], S13 = par[3], S22 = par[4], S23 = par[5], S33 = par[6], gpref = par[7];
        // ---- equilibrium tables ----
        auto hcoef = [&](int k) {  // Horner coefficients z^c Z(k) of pass 2
            const double z = g.node(k), Z = Ztab[k];
            double* h = Htab + 6 * k;
            h[0] = Z; h[1] = z * Z; h[2] = z * (z * Z); h[3] = z * (z * (z * Z)); h[4] = z * (z * (z * (z * Z)));
        };
        {
            const double dz0 = g.node(0) - m.uz, dv = g.dv;
            if (gauss) {
                for (int k = t; k < n; k += MT) {
                    const double dz = g.node(k) - m.uz;
                    Ztab[k] = exp(-0.5 * S33 * dz * dz);
                    hcoef(k);
                }
                for (int pidx = t; pidx < n * n; pidx += MT) {
                    const double dx = g.node(pidx >> lg) - m.ux, dy = g.node(pidx & (n - 1)) - m.uy;
                    const double L = S13 * dx + S23 * dy;
                    const double eP = -0.5 * (S11 * dx * dx + 2.0 * S12 * dx * dy + S22 * dy * dy) - L * dz0;
                    const double eR = -L * dv;
                    if (!(fabs(eP) < 600.0 && fabs(eR) * (n - 1) < 600.0 && fabs(eP + eR * (n - 1)) < 600.0))
                        par[8] = 1.0;  // benign race: every writer stores 1
                    Ptab[pidx] = gpref * exp(eP);
                    Rtab[pidx] = exp(eR);
                }
            } else {  // Maxwellian: separable (src/moments.cpp:93-102)
                const double inv2T = 0.5 / m.T, mpref = m.rho / pow(2.0 * M_PI * m.T, 1.5);
                for (int k = t; k < n; k += MT) {
                    const double dz = g.node(k) - m.uz;
                    Ztab[k] = exp(-dz * dz * inv2T);
                    hcoef(k);
                }
                for (int pidx = t; pidx < n * n; pidx += MT) {
                    const double dx = g.node(pidx >> lg) - m.ux, dy = g.node(pidx & (n - 1)) - m.uy;
                    Ptab[pidx] = mpref * exp(-dx * dx * inv2T) * exp(-dy * dy * inv2T);
                    Rtab[pidx] = 1.0;
                }
            }
        }
        __syncthreads();
        const bool direct = par[8] != 0.0;
        // equilibrium at the 4 nodes of group idx (k1, k2 fixed, k3 .. k3+3)
        auto eq4 = [&](int k1, int k2, int k3, double (&e)[4]) {
            if (!direct) {
                const int pidx = (k1 << lg) | k2;
                const double P = Ptab[pidx], R = Rtab[pidx];
                double rk = 1.0, r = R;
#pragma unroll
                for (int b = 0; b < 7; ++b) {  // R^k3, k3 < 128
                    if (b < lg) {
                        rk = ((k3 >> b) & 1) ? rk * r : rk;
                        r *= r;
                    }
                }
                double v = P * rk;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    e[j] = v * Ztab[k3 + j];
                    v *= R;
                }
            } else {
                const double dx = g.node(k1) - m.ux, dy = g.node(k2) - m.uy;
                const double qxy = S11 * dx * dx + 2.0 * S12 * dx * dy + S22 * dy * dy, lz = 2.0 * (S13 * dx + S23 * dy);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double dz = g.node(k3 + j) - m.uz;
                    e[j] = gpref * exp(-0.5 * (qxy + dz * (lz + S33 * dz)));
                }
            }
        };
        SP_MARK(1);
        // ---- pass 2: coupling matrix of the equilibrium (14 monomial moments) ----
        const double mom3[3] = {m.rho * m.ux, m.rho * m.uy, m.rho * m.uz};
        const double uc[3] = {mom3[0] / m.rho, mom3[1] / m.rho, mom3[2] / m.rho};
        {
            double M[14];
#pragma unroll
            for (int k = 0; k < 14; ++k) M[k] = 0.0;
            if (!direct) {
                // Per pencil, sum_k3 z^c e = P sum_k3 (z^c Z)(k3) R^k3: five polynomials in R by
                // Horner (5 FMA per node), PB pencils per thread sharing the coefficient loads.
                constexpr int PB = MINB >= 3 ? 2 : 4;  // register budget
                const int np = n << lg;
                for (int pb = t; pb < np; pb += PB * MT) {
                    double R4[PB], h[PB][5];
#pragma unroll
                    for (int u = 0; u < PB; ++u) {
                        const int pidx = pb + u * MT;
                        R4[u] = pidx < np ? Rtab[pidx] : 0.0;
#pragma unroll
                        for (int c = 0; c < 5; ++c) h[u][c] = 0.0;
                    }
#pragma unroll 4
                    for (int k3 = n - 1; k3 >= 0; --k3) {
                        const double2 a01 = *reinterpret_cast<const double2*>(Htab + 6 * k3);
                        const double2 a23 = *reinterpret_cast<const double2*>(Htab + 6 * k3 + 2);
                        const double a4 = Htab[6 * k3 + 4];
#pragma unroll
                        for (int u = 0; u < PB; ++u) {
                            h[u][0] = fma(h[u][0], R4[u], a01.x);
                            h[u][1] = fma(h[u][1], R4[u], a01.y);
                            h[u][2] = fma(h[u][2], R4[u], a23.x);
                            h[u][3] = fma(h[u][3], R4[u], a23.y);
                            h[u][4] = fma(h[u][4], R4[u], a4);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < PB; ++u) {
                        const int pidx = pb + u * MT;
                        if (pidx < np) {
                            const double P = Ptab[pidx];
                            acc14(M, g.node(pidx >> lg), g.node(pidx & (n - 1)), P * h[u][0], P * h[u][1], P * h[u][2],
                                  P * h[u][3], P * h[u][4]);
                        }
                    }
                }
            } else
#pragma unroll kStageU2
            for (int q = t; q < ngroups; q += MT) {
                const int idx = 4 * q;
                const int k1 = idx >> (2 * lg), k2 = (idx >> lg) & (n - 1), k3 = idx & (n - 1);
                double e[4];
                eq4(k1, k2, k3, e);
                double m0 = 0, m1 = 0, m2 = 0, m3 = 0, m4 = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const double z = g.node(k3 + j), zz = z * z;
                    m0 += e[j];
                    m1 += z * e[j];
                    m2 += zz * e[j];
                    m3 += zz * (z * e[j]);
                    m4 += zz * (zz * e[j]);
                }
                acc14(M, g.node(k1), g.node(k2), m0, m1, m2, m3, m4);
            }
            block_reduce(M, 14);
        }
        SP_MARK(2);
        if (t == 0) {
            double Mm[14], Amat[25];
            for (int k = 0; k < 14; ++k) Mm[k] = par[16 + k];
            coupling_from_monomials(Mm, uc, g.dvk, Amat);
            const double rhs[5] = {m.rho, mom3[0], mom3[1], mom3[2], 2.0 * energy_of(m)};
            double x[5];
            const bool ok = solve5(Amat, rhs, x);
            for (int k = 0; k < 5; ++k) par[9 + k] = x[k];
            st = ok ? HK_OK : HK_DEGENERATE;
            if (info) info[cell] = st | (fallback << 8);
            par[14] = st;
        }
        __syncthreads();
        SP_MARK(3);
        if ((int)par[14] == HK_OK) {
            const double x[5] = {par[9], par[10], par[11], par[12], par[13]};
            const double wf = eps / (eps + A), wg = A / (eps + A);
            if (!direct) {  // (Z, Z Q) per k3, Q = cz (x3 + x4 cz)
                for (int k = t; k < n; k += MT) {
                    const double cz = g.node(k) - uc[2], Z = Ztab[k];
                    ZQ[zq_slot(k)] = make_double2(Z, Z * (cz * (x[3] + x[4] * cz)));
                }
                __syncthreads();
            }
            // ---- pass 3: out = wf f + wg G (x0 + x.c + x4 |c|^2) ----
            // Groups in reverse: the planes pass 1 loaded last are re-read first,
            // while they are most likely still in L2 (config 3: 9.91 -> 9.76 ms;
            // keeping the first 11 planes in shared memory instead cost 0.5 ms).
#pragma unroll kStageU3
            for (int qb = ((ngroups - 1) / MT) * MT; qb >= 0; qb -= MT) {
                const int q = qb + t;
                if (q >= ngroups) continue;
                const int idx = 4 * q;
                const int k1 = idx >> (2 * lg), k2 = (idx >> lg) & (n - 1), k3 = idx & (n - 1);
                const double vx = g.node(k1), vy = g.node(k2);
                double2 fa, fb;
                if constexpr (ACC) {  // f_acc parked in out by pass 1 (other threads: the solve barrier orders it)
                    fa = *reinterpret_cast<const double2*>(oc + idx);
                    fb = *reinterpret_cast<const double2*>(oc + idx + 2);
                } else {
                    fa = ldg2_hint(fc + idx, pol_first);
                    fb = ldg2_hint(fc + idx + 2, pol_first);
                }
                const double fv[4] = {fa.x, fa.y, fb.x, fb.y};
                const double cx = vx - uc[0], cy = vy - uc[1];
                const double pxy = x[0] + x[1] * cx + x[2] * cy + x[4] * (cx * cx + cy * cy);
                double o[4];
                if (!direct) {  // wg e (pxy + Q) = (wg P R^k3) (Z pxy + Z Q)
                    const int pidx = (k1 << lg) | k2;
                    const double R = Rtab[pidx];
                    double rk = 1.0, r = R;
#pragma unroll
                    for (int b = 0; b < 7; ++b) {  // R^k3, k3 < 128
                        if (b < lg) {
                            rk = ((k3 >> b) & 1) ? rk * r : rk;
                            r *= r;
                        }
                    }
                    double v = (wg * Ptab[pidx]) * rk;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const double2 zq = ZQ[zq_slot(k3 + j)];
                        o[j] = fma(wf, fv[j], v * fma(zq.x, pxy, zq.y));
                        v *= R;
                    }
                } else {
                    double e[4];
                    eq4(k1, k2, k3, e);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const double cz = g.node(k3 + j) - uc[2];
                        o[j] = wf * fv[j] + wg * (e[j] * (pxy + cz * (x[3] + x[4] * cz)));
                    }
                }
                st2_hint(oc + idx, make_double2(o[0], o[1]), pol_first);
                st2_hint(oc + idx + 2, make_double2(o[2], o[3]), pol_first);
                if (k1_out) {  // fused K1 of the IMEX step: k1 = (Y - f) / a11
                    double* kc = k1_out + cell * nb + idx;
                    st2_hint(kc, make_double2((o[0] - fv[0]) * k1_scale, (o[1] - fv[1]) * k1_scale), pol_first);
                    st2_hint(kc + 2, make_double2((o[2] - fv[2]) * k1_scale, (o[3] - fv[3]) * k1_scale), pol_first);
                }
            }
        }
        __syncthreads();  // tables / par reused by the next cell
        SP_MARK(4);
    }
#if HK_STAGE_PROF
    if (t == 0)
        for (int q = 0; q < 5; ++q) atomicAdd(&g_stage_prof[q], (unsigned long long)sp[q]);
#endif
#undef SP_MARK
}

__global__ void k1_kernel(int64_t count, double* __restrict__ k1, const double* __restrict__ y,
                          const double* __restrict__ f, double scale) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        k1[i] = (y[i] - f[i]) * scale;
}

bool warp_path(int n) { return n >= 8 && n <= 64 && (n & (n - 1)) == 0; }
int log2i(int n) {
    int l = 0;
    while ((1 << l) < n) ++l;
    return l;
}

// ---------------------------------------------------------------------------
// Stand-alone moment operators of inc/moments.hpp:55-70 (the stage and
// residual kernels fuse them; these are the drop-ins for callers that use them
// one at a time).  One CTA per cell.
// ---------------------------------------------------------------------------
// Eigen::LLT test, determinant and inverse of a 3x3 SPD candidate as the stage
// kernel does them (src/moments.cpp:128-138).  par[0..8] = inverse (row-major),
// par[9] = rho / sqrt((2 pi)^3 det).  Returns false when LLT fails.
__device__ bool gaussian_params(const double tc[9], double rho, double* par) {
    double l[9] = {0};
    for (int k = 0; k < 3; ++k) {
        double x = tc[3 * k + k];
        for (int j = 0; j < k; ++j) x -= l[3 * k + j] * l[3 * k + j];
        if (!(x > 0.0)) return false;
        l[3 * k + k] = sqrt(x);
        for (int i = k + 1; i < 3; ++i) {
            double y = tc[3 * i + k];
            for (int j = 0; j < k; ++j) y -= l[3 * i + j] * l[3 * k + j];
            l[3 * i + k] = y / l[3 * k + k];
        }
    }
    const double* q = tc;
    const double c00 = q[4] * q[8] - q[5] * q[7], c01 = q[5] * q[6] - q[3] * q[8], c02 = q[3] * q[7] - q[4] * q[6];
    const double det = q[0] * (q[4] * q[8] - q[5] * q[7]) - q[1] * (q[3] * q[8] - q[5] * q[6]) +
                       q[2] * (q[3] * q[7] - q[4] * q[6]);
    const double id = 1.0 / (q[0] * c00 + q[1] * c01 + q[2] * c02);
    par[0] = c00 * id; par[1] = (q[2] * q[7] - q[1] * q[8]) * id; par[2] = (q[1] * q[5] - q[2] * q[4]) * id;
    par[3] = c01 * id; par[4] = (q[0] * q[8] - q[2] * q[6]) * id; par[5] = (q[2] * q[3] - q[0] * q[5]) * id;
    par[6] = c02 * id; par[7] = (q[1] * q[6] - q[0] * q[7]) * id; par[8] = (q[0] * q[4] - q[1] * q[3]) * id;
    par[9] = rho / sqrt(pow(2.0 * M_PI, 3) * det);
    return true;
}

// anisotropic_gaussian (src/moments.cpp:120-157): mom[cell] = (rho, u, T),
// theta[cell] = stress tensor (3x3 row-major); fallback[cell] = 1 when the
// corrected tensor fails LLT (the Maxwellian is written instead).
__global__ void __launch_bounds__(NT) gaussian_kernel(const double* __restrict__ mom, const double* __restrict__ theta,
                                                      double beta, int64_t ncells, VGrid g, double* __restrict__ out,
                                                      int* __restrict__ fallback) {
    __shared__ double ex[128], ey[128], ez[128];
    __shared__ double par[11];
    const int n = g.n, nb = n * n * n;
    for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
        const Mom m{mom[cell * 5], mom[cell * 5 + 1], mom[cell * 5 + 2], mom[cell * 5 + 3], mom[cell * 5 + 4]};
        if (threadIdx.x == 0) {
            double tc[9];
            const double iso = (1.0 - beta) * m.T;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) tc[3 * i + j] = (i == j ? iso : 0.0) + beta * theta[cell * 9 + 3 * i + j];
            par[10] = gaussian_params(tc, m.rho, par) ? 1.0 : 0.0;
            if (fallback) fallback[cell] = par[10] != 0.0 ? 0 : 1;
        }
        __syncthreads();
        double* o = out + cell * nb;
        if (par[10] != 0.0) {
            for (int idx = threadIdx.x; idx < nb; idx += NT) {
                const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
                const double dx = g.node(k1) - m.ux, dy = g.node(k2) - m.uy, dz = g.node(k3) - m.uz;
                const double qxy = par[0] * dx * dx + 2.0 * par[1] * dx * dy + par[4] * dy * dy;
                const double lz = 2.0 * (par[2] * dx + par[5] * dy);
                o[idx] = par[9] * exp(-0.5 * (qxy + dz * (lz + par[8] * dz)));
            }
        } else {
            const double pref = maxwell_factors(m, g, ex, ey, ez);
            for (int idx = threadIdx.x; idx < nb; idx += NT) {
                const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
                o[idx] = pref * ex[k1] * ey[k2] * ez[k3];
            }
        }
        __syncthreads();
    }
}

// match_moments (src/moments.cpp:225-246), in place: target[cell] = (rho,
// momentum x/y/z, energy); status HK_DEGENERATE when the system is singular
// (f untouched).
__global__ void __launch_bounds__(NT) match_kernel(double* __restrict__ f, const double* __restrict__ target,
                                                   int64_t ncells, VGrid g, int* __restrict__ status) {
    __shared__ double scratch[8 * 25];
    __shared__ double par[6];
    const int n = g.n, nb = n * n * n;
    for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
        double* fc = f + cell * nb;
        const double* tg = target + cell * 5;
        const double uc[3] = {tg[1] / tg[0], tg[2] / tg[0], tg[3] / tg[0]};
        double A[25];
        coupling(g, uc, [&](int idx, double, double, double) { return fc[idx]; }, A, scratch);
        if (threadIdx.x == 0) {
            const double rhs[5] = {tg[0], tg[1], tg[2], tg[3], 2.0 * tg[4]};
            double x[5];
            const bool ok = solve5(A, rhs, x);
            for (int k = 0; k < 5; ++k) par[k] = x[k];
            par[5] = ok ? 1.0 : 0.0;
            if (status) status[cell] = ok ? HK_OK : HK_DEGENERATE;
        }
        __syncthreads();
        if (par[5] != 0.0) {
            const double x[5] = {par[0], par[1], par[2], par[3], par[4]};
            for (int idx = threadIdx.x; idx < nb; idx += NT) {
                const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
                fc[idx] *= quad_factor(x, g.node(k1), g.node(k2), g.node(k3), uc);
            }
        }
        __syncthreads();
    }
}

// remove_invariant_moments (src/moments.cpp:248-267), in place on q with the
// weight w and centre uc[cell]; HK_DEGENERATE when the coupling is singular.
__global__ void __launch_bounds__(NT) remove_invariants_kernel(double* __restrict__ q, const double* __restrict__ w,
                                                               const double* __restrict__ ucs, int64_t ncells, VGrid g,
                                                               int* __restrict__ status) {
    __shared__ double scratch[8 * 25];
    __shared__ double par[6];
    const int n = g.n, nb = n * n * n;
    for (int64_t cell = blockIdx.x; cell < ncells; cell += gridDim.x) {
        double* qc = q + cell * nb;
        const double* wc = w + cell * nb;
        const double uc[3] = {ucs[cell * 3], ucs[cell * 3 + 1], ucs[cell * 3 + 2]};
        double B[25];
        coupling(g, uc, [&](int idx, double, double, double) { return wc[idx]; }, B, scratch);
        double inv[5] = {0, 0, 0, 0, 0};
        for (int idx = threadIdx.x; idx < nb; idx += NT) {
            const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
            const double vx = g.node(k1), vy = g.node(k2), vz = g.node(k3);
            const double o = qc[idx];
            inv[0] += o;
            inv[1] += vx * o;
            inv[2] += vy * o;
            inv[3] += vz * o;
            inv[4] += (vx * vx + vy * vy + vz * vz) * o;
        }
        block_sum<5>(inv, scratch);
        if (threadIdx.x == 0) {
            double rhs[5], y[5];
            for (int k = 0; k < 5; ++k) rhs[k] = inv[k] * g.dvk;
            const bool ok = solve5(B, rhs, y);
            for (int k = 0; k < 5; ++k) par[k] = y[k];
            par[5] = ok ? 1.0 : 0.0;
            if (status) status[cell] = ok ? HK_OK : HK_DEGENERATE;
        }
        __syncthreads();
        if (par[5] != 0.0) {
            const double y[5] = {par[0], par[1], par[2], par[3], par[4]};
            for (int idx = threadIdx.x; idx < nb; idx += NT) {
                const int k3 = idx % n, k2 = (idx / n) % n, k1 = idx / (n * n);
                qc[idx] -= quad_factor(y, g.node(k1), g.node(k2), g.node(k3), uc) * wc[idx];
            }
        }
        __syncthreads();
    }
}

int grid_for(hk_ctx ctx, int64_t ncells) {
    const int64_t cap = int64_t(ctx->sm_count) * 8;
    return int(ncells < cap ? ncells : cap);
}

}  // namespace

int moments_launch(hk_ctx ctx, int n, double vmax, const double* f, int64_t ncells, double* mom, double* sigma,
                   double* real, double* l1, int* status, const int64_t* src_idx,
                   const int* count_dev) {
    if (ncells <= 0) return HK_OK;
    if (n < 2 || n > 128) return fail(ctx, HK_UNSUPPORTED, "moments: 2 <= n <= 128");
    // 256-thread CTAs, 2 per SM, 16 loads in flight per thread (config 3: 3.99 ms;
    // measured and removed: 512 x 1 x 16, 256 x 4 x 8 4.72 ms, 128 x 6 x 8, 512 x 2 x 8, 256 x 3 x 8)
    if (warp_path(n)) {
        const int64_t cap = int64_t(ctx->sm_count) * 2;
        const int grid = int(ncells < cap ? ncells : cap);
        moments_cta_kernel<256, 2, 16><<<grid, 256, 0, ctx->stream>>>(f, ncells, make_vgrid(n, vmax), log2i(n), mom, sigma,
                                                                      real, l1, status, src_idx, count_dev);
    } else
        moments_kernel<<<grid_for(ctx, ncells), NT, 0, ctx->stream>>>(f, ncells, make_vgrid(n, vmax), mom, sigma, real,
                                                                      l1, status, src_idx, count_dev);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "moments kernel");
}

int maxwellian_launch(hk_ctx ctx, int n, double vmax, const double* mom, int64_t ncells, double* out, int* status,
                      const int64_t* dst_idx, const int* count_dev) {
    if (ncells <= 0) return HK_OK;
    if (n < 2 || n > 128) return fail(ctx, HK_UNSUPPORTED, "maxwellian: 2 <= n <= 128");
    maxwellian_kernel<<<grid_for(ctx, ncells), NT, 0, ctx->stream>>>(mom, ncells, make_vgrid(n, vmax), out, status,
                                                                     dst_idx, count_dev);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "maxwellian kernel");
}

size_t stage_smem(int n) { return sizeof(double) * (2 * n * n + n + 8 * 16 + 32 + 2 * n + 6 * n + 2 * n); }

bool stage_acc_supported(int n) { return warp_path(n); }

int stage_acc_launch(hk_ctx ctx, bool esbgk, int n, double vmax, const double* f, const double* q1, const double* k1,
                     double cq, double ck, double* out, int64_t ncells, double a, const double* eps_cell, double beta,
                     double coeff, int* info) {
    if (ncells <= 0) return HK_OK;
    if (!stage_acc_supported(n)) return fail(ctx, HK_UNSUPPORTED, "fused stage: n a power of two >= 8");
    const VGrid g = make_vgrid(n, vmax);
    const int64_t cap = int64_t(ctx->sm_count) * 2;
    const int grid = int(ncells < cap ? ncells : cap);
    const size_t smem = stage_smem(n);
    auto kern = esbgk ? stage_cta_kernel<true, 256, 2, true> : stage_cta_kernel<false, 256, 2, true>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 256, smem, ctx->stream>>>(f, out, ncells, g, log2i(n), a, eps_cell, 0.0, beta, coeff, info, nullptr,
                                           nullptr, 0.0, AccIn{q1, k1, cq, ck});
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "fused stage kernel");
}

int stage_launch(hk_ctx ctx, bool esbgk, int n, double vmax, const double* fin, double* out, int64_t ncells, double a,
                 const double* eps_cell, double eps_scalar, double beta, double coeff, int* info, double* mom_out,
                 double* k1_out, double k1_scale) {
    if (ncells <= 0) return HK_OK;
    if (n < 2 || n > 128) return fail(ctx, HK_UNSUPPORTED, "stage: 2 <= n <= 128");
    const VGrid g = make_vgrid(n, vmax);
    if (warp_path(n)) {
        // 256-thread CTAs, 2 per SM (config 3, L2 hints, register solve5: 9.9 ms; measured and
        // removed: 3 per SM 10.9, 128-thread CTAs 5 / 6 per SM 10.2 / 10.4)
        const int64_t cap = int64_t(ctx->sm_count) * 2;
        const int grid = int(ncells < cap ? ncells : cap);
        const size_t smem = stage_smem(n);
        auto kern = esbgk ? stage_cta_kernel<true, 256, 2> : stage_cta_kernel<false, 256, 2>;
        const int mt = 256;
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, mt, smem, ctx->stream>>>(fin, out, ncells, g, log2i(n), a, eps_cell, eps_scalar, beta, coeff, info,
                                              mom_out, k1_out, k1_scale, AccIn{});
#if HK_STAGE_PROF
        {
            unsigned long long h[5];
            cudaStreamSynchronize(ctx->stream);
            cudaMemcpyFromSymbol(h, g_stage_prof, sizeof h);
            const double tot = double(h[0] + h[1] + h[2] + h[3] + h[4]);
            fprintf(stderr, "[hk stage prof] pass1 %.1f%% tail1+tables %.1f%% pass2 %.1f%% solve %.1f%% pass3 %.1f%%\n",
                    100 * h[0] / tot, 100 * h[1] / tot, 100 * h[2] / tot, 100 * h[3] / tot, 100 * h[4] / tot);
            const unsigned long long z[5] = {0, 0, 0, 0, 0};
            cudaMemcpyToSymbol(g_stage_prof, z, sizeof z);
        }
#endif
        ctx->launches++;
        return check_cuda(ctx, cudaGetLastError(), "stage kernel");
    } else if (esbgk)
        stage_kernel<true><<<grid_for(ctx, ncells), NT, 0, ctx->stream>>>(fin, out, ncells, g, a, eps_cell, eps_scalar,
                                                                          beta, coeff, info, mom_out);
    else
        stage_kernel<false><<<grid_for(ctx, ncells), NT, 0, ctx->stream>>>(fin, out, ncells, g, a, eps_cell, eps_scalar,
                                                                           beta, coeff, info, mom_out);
    ctx->launches++;
    int st = check_cuda(ctx, cudaGetLastError(), "stage kernel");
    if (!st && k1_out) {  // these kernels do not fuse K1
        const int64_t count = ncells * (int64_t)n * n * n;
        k1_kernel<<<unsigned(std::min<int64_t>((count + 255) / 256, int64_t(ctx->sm_count) * 16)), 256, 0, ctx->stream>>>(
            count, k1_out, out, fin, k1_scale);
        ctx->launches++;
        st = check_cuda(ctx, cudaGetLastError(), "k1 kernel");
    }
    return st;
}

int residual_finish_launch(hk_ctx ctx, int n, double vmax, const double* f, double* q, int64_t ncells, double pen_coeff,
                           int* status) {
    if (ncells <= 0) return HK_OK;
    if (warp_path(n)) {
        // one CTA per cell, two streaming passes (the coupling matrices from 1-D sums)
        const int64_t cap = int64_t(ctx->sm_count) * HK_RES_MINB;
        const int grid = int(ncells < cap ? ncells : cap);
        residual_cta_kernel<HK_RES_MT, HK_RES_MINB><<<grid, HK_RES_MT, 0, ctx->stream>>>(f, q, ncells, make_vgrid(n, vmax),
                                                                                      log2i(n), pen_coeff, status);
    } else
        residual_finish_kernel<<<grid_for(ctx, ncells), NT, 0, ctx->stream>>>(f, q, ncells, make_vgrid(n, vmax),
                                                                              pen_coeff, status);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "residual kernel");
}

int gaussian_launch(hk_ctx ctx, int n, double vmax, const double* mom, const double* theta, double beta,
                    int64_t ncells, double* out, int* fallback) {
    if (ncells <= 0) return HK_OK;
    if (n < 2 || n > 128) return fail(ctx, HK_UNSUPPORTED, "anisotropic_gaussian: 2 <= n <= 128");
    gaussian_kernel<<<grid_for(ctx, ncells), NT, 0, ctx->stream>>>(mom, theta, beta, ncells, make_vgrid(n, vmax), out,
                                                                   fallback);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "gaussian kernel");
}

int match_launch(hk_ctx ctx, int n, double vmax, double* f, const double* target, int64_t ncells, int* status) {
    if (ncells <= 0) return HK_OK;
    if (n < 2 || n > 128) return fail(ctx, HK_UNSUPPORTED, "match_moments: 2 <= n <= 128");
    match_kernel<<<grid_for(ctx, ncells), NT, 0, ctx->stream>>>(f, target, ncells, make_vgrid(n, vmax), status);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "match kernel");
}

int remove_invariants_launch(hk_ctx ctx, int n, double vmax, double* q, const double* w, const double* uc,
                             int64_t ncells, int* status) {
    if (ncells <= 0) return HK_OK;
    if (n < 2 || n > 128) return fail(ctx, HK_UNSUPPORTED, "remove_invariant_moments: 2 <= n <= 128");
    remove_invariants_kernel<<<grid_for(ctx, ncells), NT, 0, ctx->stream>>>(q, w, uc, ncells, make_vgrid(n, vmax),
                                                                            status);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "remove-invariants kernel");
}

}  // namespace hk
