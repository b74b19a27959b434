// hk_transport.cu — CWENO3 upwind kinetic transport sweep, y-marching
// (kinetic_transport_rhs_cell / _periodic, src/transport.cpp:12-66; cweno3,
// src/euler.cpp:10-40).  Compiled with FMA contraction (hk_field.cu, which
// keeps the per-node kernel and the classifier bitwise to the reference, is
// not); results agree with the reference to ~1e-15 relative.
#include <cstdlib>

#include "hk_cells.cuh"
#include "hk_common.cuh"

namespace hk {

namespace {

// Face values of the CWENO3 reconstruction (src/euler.cpp:10-40) with the
// three nonlinear weights normalised through ONE reciprocal:
//   a_k = c_k / D_k^2  ->  w_k = c_k P_k / sum_m c_m P_m,  P_k = prod_{m != k} D_m^2
// (same values as the reference's three divisions up to rounding).
// 1/x for the normalisation of the nonlinear weights (x >= eps^2 (...) > 0,
// never denormal): the MUFU seed refined by two Newton steps (~1 ulp), without
// the IEEE division's slow-path branch.
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

// One face only (the upwind one), the same CWENO3 value in fewer operations:
// with the weights summing to one, c0 = uc - a_c c / 12, so
//   right = uc + (1/S) [ (p_l s_l + p_r s_r) / 2 + p_c (b / 2 + c / 6) ]
//   left  = uc + (1/S) [-(p_l s_l + p_r s_r) / 2 + p_c (c / 6 - b / 2) ]
// with p = 4 x (the weights' numerators above) and S their sum (~31 instead
// of ~45 fp64 operations per face).
template <bool RIGHT>
__device__ __forceinline__ double cweno3_face(double um, double uc, double up, double eps) {
    const double sl = uc - um, sr = up - uc;
    const double b = 0.5 * (up - um);
    const double c = sr - sl;  // up - 2 uc + um
    const double dl = fma(sl, sl, eps), dr = fma(sr, sr, eps), dc = fma((13.0 / 3.0) * c, c, fma(b, b, eps));
    const double l2 = dl * dl, r2 = dr * dr, c2 = dc * dc;
    const double pl = c2 * r2, pr = l2 * c2, pc = (l2 + l2) * r2;
    const double inv = rcp_nr(pl + pc + pr);
    const double side = 0.5 * fma(pl, sl, pr * sr);
    const double mid = RIGHT ? fma(c, 1.0 / 6.0, 0.5 * b) : fma(c, 1.0 / 6.0, -0.5 * b);
    return fma(inv, RIGHT ? fma(pc, mid, side) : fma(pc, mid, -side), uc);
}

// Transport sweep (production path): lanes march the rows j = 0 .. ny-1 with
// the y stencil as a 5-value sliding window in registers (one new load per
// step); the upwind face computed at step j is the minus face of step j+1, so
// a step costs one y reconstruction instead of two.  (A thread-per-column
// variant with x neighbours through L1 was measured slower and removed.)
// Lane-per-column sweep: lane l of a warp owns column i = 28 b - 2 + l for
// NPT consecutive velocity nodes and marches down the rows.  The x neighbours' centre values come from the neighbouring lanes
// (shuffles, no loads), and the x minus face of lane l is lane l-1's plus
// face, so a row costs ONE x and ONE y reconstruction per node (2 instead of
// 3); lanes 0, 1, 30, 31 are halo columns (no output).
constexpr int TL_OUT = 28;

// STAGED: the rows the march needs next (the y-field's row j+3 and the
// fused modes' cell-local row j+1) arrive through a ring of shared-memory
// slots filled RING_ROWS - 1 rows ahead with cp.async (L2 -> SMEM, no
// registers held, L1 bypassed), four threads per cell so a warp's copy spans
// 8 cells x 64 B instead of 32 cells x 16 B.  One CTA barrier per row.
constexpr int RING_ROWS = 8, RING_CS = 10;  // slots (a power of two); doubles per cell row (8 + pad: conflict-free 16 B reads)
template <int MODE, int NPT, bool MASK = false, bool STAGED = false>
__global__ void __launch_bounds__(128) transport_lanes_kernel(TransportParams p, int lg, const double* __restrict__ f,
                                                              double* __restrict__ out, const double* __restrict__ lh,
                                                              const double* __restrict__ rh, FinalCombine fc) {
    static_assert(NPT == 2, "double2 node pairs");
    static_assert(!(STAGED && (MASK || MODE == 1)), "staged: unmasked, one cell-local input");
    __shared__ __align__(16) double ringS[STAGED ? RING_ROWS * 32 * RING_CS : 2];
    __shared__ __align__(16) double ringF[STAGED && MODE ? RING_ROWS * 32 * RING_CS : 2];
    extern __shared__ uint8_t act_s[];  // this strip's row activity (MASK: p.row_act)
    if (MASK) {
        for (int t = threadIdx.x; t < p.ny; t += blockDim.x) act_s[t] = p.row_act[(int64_t)blockIdx.x * p.ny + t];
        __syncthreads();
    }
    const int n = p.n;
    const int64_t nb = (int64_t)n * n * n;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t grp = (int64_t)blockIdx.y * (blockDim.x >> 5) + w;
    if (grp * NPT >= nb) return;  // warp-uniform
    const int64_t idx = grp * NPT;
    const int k1 = (int)(idx >> (2 * lg)), k2 = (int)((idx >> lg) & (n - 1)), k3 = (int)(idx & (n - 1));
    const int i = blockIdx.x * TL_OUT - 2 + lane;
    const bool outlane = lane >= 2 && lane < 2 + TL_OUT && i < p.nx;
    const double dv = 2.0 * p.vmax / n;
    const double vx = -p.vmax + (k1 + 0.5) * dv, vy = -p.vmax + (k2 + 0.5) * dv;
    const double inv_dx = 1.0 / p.dx, inv_dy = 1.0 / p.dy, eps = p.eps_weno;
    const int xh = p.x_halo > 0 ? p.x_halo : 0;
    const int nxi = p.nx + 2 * xh;
    const int ny = p.ny;
    // a column's source: interior (periodic wrap), halo buffer, or ghost column
    auto col_src = [&](int ii, const double*& colbase, int64_t& rowstride) {
        if (p.x_halo < 0) {
            ii = ii < -2 ? -2 : (ii > p.nx + 1 ? p.nx + 1 : ii);  // lanes past the halo are never used
            if (ii < 0) { colbase = lh + (int64_t)(p.lnx + ii) * nb; rowstride = (int64_t)p.lnx * nb; }
            else if (ii >= p.nx) { colbase = rh + (int64_t)(ii - p.nx) * nb; rowstride = (int64_t)p.rnx * nb; }
            else { colbase = f + (int64_t)ii * nb; rowstride = (int64_t)nxi * nb; }
        } else if (p.x_halo == 0) {
            ii = ((ii % p.nx) + p.nx) % p.nx;
            colbase = f + (int64_t)ii * nb;
            rowstride = (int64_t)nxi * nb;
        } else {
            ii = ii < -xh ? -xh : (ii > p.nx + xh - 1 ? p.nx + xh - 1 : ii);
            colbase = f + (int64_t)(ii + xh) * nb;
            rowstride = (int64_t)nxi * nb;
        }
    };
    const double* colbase;
    int64_t rowstride;
    col_src(i, colbase, rowstride);
    colbase += idx;
    // optional batch-resident input (periodic x only): a cell with in_pos >= 0 is read
    // from its batch row instead of the dense field
    const int iw = ((i % p.nx) + p.nx) % p.nx;
    auto ld = [&](int jj) -> double2 {
        jj = jj < 0 ? jj + ny : (jj >= ny ? jj - ny : jj);
        if (p.in_pos) {
            const int64_t c = (int64_t)jj * p.nx + iw;
            const int bb = __ldg(p.in_pos + c);
            const double* src = bb >= 0 ? p.in_batch + (int64_t)bb * nb + idx : f + c * nb + idx;
            return __ldg(reinterpret_cast<const double2*>(src));
        }
        return __ldg(reinterpret_cast<const double2*>(colbase + (int64_t)jj * rowstride));
    };
    // STAGED loader role: thread t copies 16 B (nodes idx0 + 2 h, h = t & 3) of cell lc = t >> 2
    const int lc = threadIdx.x >> 2, lh4 = threadIdx.x & 3;
    const int64_t idx0 = (int64_t)blockIdx.y * 8;
    const double* lbase = nullptr;
    int64_t lrs = 0;
    const int li = blockIdx.x * TL_OUT - 2 + lc;
    const bool lfin = STAGED && MODE && lc >= 2 && lc < 2 + TL_OUT && li < p.nx;
    // loader cursors (advanced one row per issue): y row it + 3 (periodic), cell-local row it + 1
    const double *lsrc = nullptr, *lwrap = nullptr, *fsrc = nullptr;
    int64_t fstride = 0;
    int jnext = 3 % (ny > 0 ? ny : 1);
    if constexpr (STAGED) {
        col_src(li, lbase, lrs);
        lbase += idx0 + 2 * lh4;
        lsrc = lbase + (int64_t)jnext * lrs;
        lwrap = lbase;
        if (MODE) {
            fstride = (int64_t)p.nx * nb;
            fsrc = fc.f + ((int64_t)p.nx + li) * nb + idx0 + 2 * lh4;
        }
    }
    const uint32_t lsm = smem_u32(&ringS[lc * RING_CS + 2 * lh4]), lsmf = smem_u32(&ringF[lc * RING_CS + 2 * lh4]);
    constexpr uint32_t SLOT_B = 32 * RING_CS * sizeof(double);
    auto issue = [&](int it) {  // ring slot it % RING_ROWS <- y row it + 3 and cell-local row it + 1
        if (it < ny) {
            const uint32_t so = (it & (RING_ROWS - 1)) * SLOT_B;
            cp_async16(lsm + so, lsrc);
            if (++jnext == ny) {
                jnext = 0;
                lsrc = lwrap;
            } else {
                lsrc += lrs;
            }
            if (lfin && it + 1 < ny) cp_async16(lsmf + so, fsrc);
            fsrc += fstride;
        }
        cp_async_commit();
    };
    if constexpr (STAGED)
        for (int it = 0; it < RING_ROWS - 1; ++it) issue(it);
    auto sh_up = [&](double v, int d) { return __shfl_up_sync(0xffffffffu, v, d); };
    auto sh_dn = [&](double v, int d) { return __shfl_down_sync(0xffffffffu, v, d); };
    double2 w0 = ld(-2), w1 = ld(-1), w2 = ld(0), w3 = ld(1), w4 = ld(2);
    const bool ypos = vy > 0.0, xpos = vx > 0.0;
    auto yface = [&](double a, double b, double c, double d, double e) -> double {  // new upwind y face
        return ypos ? cweno3_face<true>(b, c, d, eps) : cweno3_face<false>(c, d, e, eps);
    };
    double fyp[2];
    if (ypos) {
        fyp[0] = cweno3_face<true>(w0.x, w1.x, w2.x, eps);
        fyp[1] = cweno3_face<true>(w0.y, w1.y, w2.y, eps);
    } else {
        fyp[0] = cweno3_face<false>(w1.x, w2.x, w3.x, eps);
        fyp[1] = cweno3_face<false>(w1.y, w2.y, w3.y, eps);
    }
    double2 nw4 = make_double2(0, 0), nf0 = nw4, nf1 = nw4, nf2 = nw4;
    // the cell-local inputs of the fused modes, loaded one row ahead (f / G is
    // read and rewritten by this lane only: plain loads, in place)
    auto fin_loads = [&](int jj, double2& a, double2& b, double2& c) {
        const int64_t o = ((int64_t)jj * p.nx + i) * nb + idx;
        a = *reinterpret_cast<const double2*>(fc.f + o);
        if constexpr (MODE == 1) {
            b = __ldg(reinterpret_cast<const double2*>(fc.q1 + o));
            c = __ldg(reinterpret_cast<const double2*>(fc.k1 + o));
        }
    };
    if (MODE && outlane) fin_loads(0, nf0, nf1, nf2);
    // row activity under the optional mask (warp-uniform): a row is computed
    // when one of the strip's output cells is masked in; its y face also when
    // the next row is (the face is shared)
    auto row_active = [&](int jj) -> bool { return !MASK || act_s[jj] != 0; };
    bool act = row_active(0), act_next = ny > 1 ? row_active(1) : false;
    for (int j = 0; j < ny; ++j) {
        if (j > 0) {
            w0 = w1; w1 = w2; w2 = w3; w3 = w4;
            w4 = nw4;
        }
        const double2 cf = nf0, cq = nf1, ck = nf2;
        if constexpr (STAGED) {
            cp_async_wait_group<RING_ROWS - 2>();  // this thread's copies of slot j landed
            __syncthreads();                       // everyone's; and everyone is done with slot j - 1
            issue(j + RING_ROWS - 1);              // into slot j - 1
            if (j + 1 < ny) {
                const int so = (j & (RING_ROWS - 1)) * 32 * RING_CS + lane * RING_CS + 2 * w;
                nw4 = *reinterpret_cast<const double2*>(&ringS[so]);
                if (MODE && outlane) nf0 = *reinterpret_cast<const double2*>(&ringF[so]);
            }
        } else if (j + 1 < ny) {
            nw4 = ld(j + 3);  // row j+3 = w4 of row j+1
            if (MODE && outlane) fin_loads(j + 1, nf0, nf1, nf2);
        }
        const bool act_nn = MASK && j + 2 < ny ? row_active(j + 2) : false;
        if (MASK && !act && !act_next) {  // nothing here, and the next row does not need this row's face
            if (!act_nn) {
                // a run of inactive rows: jump to L = (next active row) - 1, whose face
                // is the first one needed, instead of streaming the rows between
                int r = j + 3;
                while (r < ny && !row_active(r)) ++r;
                if (r >= ny) break;  // no active row left in this strip
                const int L = r - 1;
                if (L > j + 2) {  // otherwise the plain march gets there as cheaply
                    w1 = ld(L - 2); w2 = ld(L - 1); w3 = ld(L); w4 = ld(L + 1); nw4 = ld(L + 2);
                    j = L - 1;
                    act = false;
                    act_next = true;
                    continue;
                }
            }
            act = act_next;
            act_next = act_nn;
            continue;
        }
        const double c[2] = {w2.x, w2.y};
        double fy[2], fx[2];
        fy[0] = yface(w0.x, w1.x, w2.x, w3.x, w4.x);
        fy[1] = yface(w0.y, w1.y, w2.y, w3.y, w4.y);
        if (MASK && !act) {  // face only (the minus face of the next, active row)
            fyp[0] = fy[0];
            fyp[1] = fy[1];
            act = act_next;
            act_next = act_nn;
            continue;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const double cp1 = sh_dn(c[q], 1);
            double plus;
            if (xpos) {  // right face of cell i
                const double cm1 = sh_up(c[q], 1);
                plus = cweno3_face<true>(cm1, c[q], cp1, eps);
            } else {     // left face of cell i+1
                const double cp2 = sh_dn(c[q], 2);
                plus = cweno3_face<false>(c[q], cp1, cp2, eps);
            }
            const double minus = sh_up(plus, 1);
            fx[q] = vx * (plus - minus);
        }
        if (outlane) {
            const int64_t o = ((int64_t)j * p.nx + i) * nb + idx;
            double tr[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) tr[q] = -fx[q] * inv_dx - vy * (fy[q] - fyp[q]) * inv_dy;
            if constexpr (MODE == 0) {
                if (p.out_pos) {  // compact output: the batch row of this cell, if any
                    const int b = p.out_pos[(int64_t)j * p.nx + i];
                    if (b >= 0) *reinterpret_cast<double2*>(out + (int64_t)b * nb + idx) = make_double2(tr[0], tr[1]);
                } else {
                    *reinterpret_cast<double2*>(out + o) = make_double2(tr[0], tr[1]);
                }
            } else if constexpr (MODE == 2) {  // T(Y1): f_acc and G (FinalCombine)
                const int64_t cell = (int64_t)j * p.nx + i;
                const double ie = fc.res ? 1.0 / fc.eps[cell] : 0.0;
                const double fv[2] = {cf.x, cf.y}, y1[2] = {w2.x, w2.y};
                const double cy = fc.w_im1 / fc.a_im11;
                double fa2[2], g2[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const double q1 = fc.res ? tr[q] + fc.res[o + q] * ie : tr[q];
                    const double k1 = (y1[q] - fv[q]) * fc.k1_scale;
                    fa2[q] = fv[q] + fc.dt * fc.a_ex10 * q1 + fc.a_im10 * k1;
                    g2[q] = fv[q] + (fc.dt * (fc.w_ex0 * q1) + fc.w_im0 * k1) - cy * fa2[q];
                }
                *reinterpret_cast<double2*>(fc.fa + o) = make_double2(fa2[0], fa2[1]);
                *reinterpret_cast<double2*>(fc.f + o) = make_double2(g2[0], g2[1]);
            } else if constexpr (MODE == 3) {  // T(Y2): f = G + dt w_ex1 q2 + (w_im1 / a_im11) Y2
                const int64_t cell = (int64_t)j * p.nx + i;
                const double ie = fc.res ? 1.0 / fc.eps[cell] : 0.0;
                const double gv[2] = {cf.x, cf.y}, y2[2] = {w2.x, w2.y};
                const double cy = fc.w_im1 / fc.a_im11;
                double o2[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const double q2 = fc.res ? tr[q] + fc.res[o + q] * ie : tr[q];
                    o2[q] = gv[q] + (fc.dt * (fc.w_ex1 * q2) + cy * y2[q]);
                }
                *reinterpret_cast<double2*>(fc.f + o) = make_double2(o2[0], o2[1]);
            } else {
                const int64_t cell = (int64_t)j * p.nx + i;
                const double ie = fc.res ? 1.0 / fc.eps[cell] : 0.0;
                const double fv[2] = {cf.x, cf.y}, q1[2] = {cq.x, cq.y}, k1v[2] = {ck.x, ck.y}, y2[2] = {w2.x, w2.y};
                double o2[2];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const double q2 = fc.res ? tr[q] + fc.res[o + q] * ie : tr[q];
                    const double facc = fv[q] + fc.dt * fc.a_ex10 * q1[q] + fc.a_im10 * k1v[q];
                    const double k2 = (y2[q] - facc) * (1.0 / fc.a_im11);
                    o2[q] = fv[q] + (fc.dt * (fc.w_ex0 * q1[q] + fc.w_ex1 * q2) + fc.w_im0 * k1v[q] + fc.w_im1 * k2);
                }
                *reinterpret_cast<double2*>(fc.f + o) = make_double2(o2[0], o2[1]);
            }
        }
        fyp[0] = fy[0];
        fyp[1] = fy[1];
        act = act_next;
        act_next = act_nn;
    }
    (void)k3;
}

// act[b][j] = any cell of interest in row j of output strip b (columns 28 b .. 28 b + 27).
__global__ void row_activity_kernel(int nx, int ny, const int8_t* __restrict__ mask, uint8_t* __restrict__ act) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int strips = (nx + TL_OUT - 1) / TL_OUT;
    if (k >= (int64_t)strips * ny) return;
    const int b = int(k / ny), j = int(k % ny);
    const int i1 = min(nx, (b + 1) * TL_OUT);
    uint8_t any = 0;
    for (int i = b * TL_OUT; i < i1; ++i) any |= mask[(int64_t)j * nx + i] != 0;
    act[k] = any;
}

}  // namespace

size_t transport_row_activity_bytes(int nx, int ny) { return size_t((nx + TL_OUT - 1) / TL_OUT) * size_t(ny); }

int transport_row_activity(hk_ctx ctx, int nx, int ny, const int8_t* mask, uint8_t* act) {
    const int64_t total = (int64_t)transport_row_activity_bytes(nx, ny);
    if (total <= 0) return HK_OK;
    row_activity_kernel<<<unsigned((total + 255) / 256), 256, 0, ctx->stream>>>(nx, ny, mask, act);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "row activity");
}

int transport_march_launch(hk_ctx ctx, const TransportParams& p, int lg, const double* f, double* out, const double* lh,
                           const double* rh, const FinalCombine* fin) {
    const int64_t nb = (int64_t)p.n * p.n * p.n;
    // 4 warps per CTA (measured: 2 or 8 warps per CTA, or loads two rows ahead, are slower)
    const dim3 grid(unsigned((p.nx + TL_OUT - 1) / TL_OUT), unsigned((nb / 2 + 3) / 4));
    const size_t smem = p.row_act ? size_t(p.ny) : 0;
    if (smem > 48 * 1024) return fail(ctx, HK_UNSUPPORTED, "transport: row activity needs ny <= 49152");
#ifndef HK_TR_STAGED
#define HK_TR_STAGED 1
#endif
    const bool staged = HK_TR_STAGED && nb % 8 == 0;  // grid.y * 8 == nb: every warp marches (CTA barriers)
    if (fin && fin->mode == 2) {
        if (staged) transport_lanes_kernel<2, 2, false, true><<<grid, 128, 0, ctx->stream>>>(p, lg, f, out, lh, rh, *fin);
        else transport_lanes_kernel<2, 2><<<grid, 128, 0, ctx->stream>>>(p, lg, f, out, lh, rh, *fin);
    } else if (fin && fin->mode == 3) {
        if (staged) transport_lanes_kernel<3, 2, false, true><<<grid, 128, 0, ctx->stream>>>(p, lg, f, out, lh, rh, *fin);
        else transport_lanes_kernel<3, 2><<<grid, 128, 0, ctx->stream>>>(p, lg, f, out, lh, rh, *fin);
    } else if (fin) {
        transport_lanes_kernel<1, 2><<<grid, 128, 0, ctx->stream>>>(p, lg, f, out, lh, rh, *fin);
    } else if (p.row_act) {
        transport_lanes_kernel<0, 2, true><<<grid, 128, smem, ctx->stream>>>(p, lg, f, out, lh, rh, FinalCombine{});
    } else {
        if (staged && !p.in_pos)  // the staged ring copies dense rows: batch input takes the plain march
            transport_lanes_kernel<0, 2, false, true><<<grid, 128, 0, ctx->stream>>>(p, lg, f, out, lh, rh, FinalCombine{});
        else transport_lanes_kernel<0, 2><<<grid, 128, 0, ctx->stream>>>(p, lg, f, out, lh, rh, FinalCombine{});
    }
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "transport kernel");
}

bool transport_final_supported(const TransportParams& p) {
    const int64_t nb = (int64_t)p.n * p.n * p.n;
    return (p.n & (p.n - 1)) == 0 && nb % 32 == 0 && p.ny >= 3 && (p.x_halo == 0 || p.x_halo == -2);
}

int transport_fused_launch(hk_ctx ctx, const TransportParams& p, const double* y, const FinalCombine& fc,
                           const double* lh, const double* rh) {
    if (!transport_final_supported(p)) return fail(ctx, HK_UNSUPPORTED, "fused transport: lane sweep shapes only");
    int lg = 0;
    while ((1 << lg) < p.n) ++lg;
    return transport_march_launch(ctx, p, lg, y, nullptr, lh, rh, &fc);
}

int transport_final_launch(hk_ctx ctx, const TransportParams& p, const double* y2, const FinalCombine& fc) {
    int lg = 0;
    while ((1 << lg) < p.n) ++lg;
    return transport_march_launch(ctx, p, lg, y2, nullptr, nullptr, nullptr, &fc);
}

}  // namespace hk
