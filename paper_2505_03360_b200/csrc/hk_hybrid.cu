// hk_hybrid.cu — the hybrid time step (SURVEY §8f "next" #1), sm_100a.
//
// The reference ships the per-cell pieces of its hybrid scheme but not the
// step driver (simulation.cpp is absent): regime_update (src/regime.cpp:25-52),
// convert_on_transition (:54-72), synthesize_hydro_state /
// synthesize_distribution (src/coupling.cpp:57-93), the layer-0 TVD-RK2
// (src/euler.cpp:172-181) and the PR(2,2,2) kinetic steps
// (src/boltzmann.cpp:47-110, src/esbgk.cpp:47-99).  hk_hybrid_step composes
// them as SPEC.md's run_scenario loop and PAPER.md Algorithm 1 describe
// (indicator pass -> regime update + conversion -> per-layer stage updates
// with cross-layer stencil synthesis); oracle/hk_oracle.c:hko_hybrid_step is
// the CPU statement of the same step (include/hykin_b200.h has the contract).
//
// Device layout: the distribution field stays dense [cell][n^3] (the transport
// sweep needs the spatial neighbours), but every per-cell kinetic operation
// (stage solves, penalized residual = collision, IMEX combinations) runs on a
// compact batch of the kinetic cells [K1 (ES-BGK) | K2 (Boltzmann)] gathered
// once per step, so the ~80 % layer-0 cells of config 4 cost nothing there.
// The dense field doubles as the transport input: the compact stage values
// are scattered into it, the layer-0 halo holds the frozen Maxwellians.
// Lists are built by one single-CTA ordered compaction (cell order, so the
// batch order is deterministic); the host reads the list lengths once.
// Compiled without FMA contraction: the conversions are bitwise the reference.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "hk_cells.cuh"
#include "hk_common.cuh"
#include "hk_internal.h"

namespace hk {
namespace {

constexpr int kLT = 1024;  // threads of the list kernels

struct HybCounts {
    unsigned long long bad;  // (cell << 8) | status, lowest first
    int nk_old, n1, n2, nm, n01, n10, n0;
    int n2a, n2b;  // layer-2 batch classes (ghost_x > 0): A interior, B ghost distance <= 2, C the rest
};

// Distance of column i from the slab interior when gx ghost columns pad each side (0 = interior).
__device__ __forceinline__ int ghost_dist(int i, int nx, int gx) {
    return i < gx ? gx - i : (i >= nx - gx ? i - (nx - gx) + 1 : 0);
}

__device__ void fail_at(HybCounts* c, int64_t cell, int code) {
    atomicMin(&c->bad, ((unsigned long long)cell << 8) | (unsigned)code);
}

// moments_from_conserved (src/coupling.cpp:7-13)
__device__ bool mom_from_u(const double* u, double hr, double* m) {
    if (!(u[0] > 0.0)) return false;
    const double p = (hr - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
    if (!(p > 0.0)) return false;
    m[0] = u[0];
    m[1] = u[1] / u[0];
    m[2] = u[2] / u[0];
    m[3] = 0.0;
    m[4] = p / u[0];
    return true;
}

// conserved_from_moments (src/coupling.cpp:15-22)
__device__ void u_from_mom(const double* m, double hr, double* u) {
    const double rho = m[0];
    u[0] = rho;
    u[1] = rho * m[1];
    u[2] = rho * m[2];
    const double u2 = m[1] * m[1] + m[2] * m[2] + m[3] * m[3];
    u[3] = rho * m[4] / (hr - 1.0) + 0.5 * rho * u2;
}

// Ordered block compaction: returns this thread's slot among the predicated
// threads of the chunk (running offset *base, updated for the next chunk).
__device__ int block_slot(bool pred, int* warp_tot, int* base) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    if (lane == 0) warp_tot[warp] = __popc(m);
    __syncthreads();
    if (warp == 0) {
        int v = warp_tot[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        warp_tot[32 + lane] = v;  // inclusive
    }
    __syncthreads();
    const int before = (warp ? warp_tot[32 + warp - 1] : 0) + __popc(m & ((1u << lane) - 1u));
    const int slot = *base + before;
    __syncthreads();
    if (threadIdx.x == kLT - 1) *base += warp_tot[32 + 31];
    __syncthreads();
    return slot;
}

// Pass A (t^n): the kinetic cells in cell order, pos[c] = batch index or -1.
__global__ void __launch_bounds__(kLT) list_old_kernel(int64_t cells, const int8_t* __restrict__ r,
                                                       int64_t* __restrict__ list, int* __restrict__ pos,
                                                       HybCounts* cnt) {
    __shared__ int wt[64];
    __shared__ int base;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < cells; c0 += kLT) {
        const int64_t c = c0 + threadIdx.x;
        const bool kin = c < cells && r[c] != 0;
        const int s = block_slot(kin, wt, &base);
        if (c < cells) {
            pos[c] = kin ? s : -1;
            if (kin) list[s] = c;
        }
    }
    if (threadIdx.x == 0) cnt->nk_old = base;
}

// Hydro view at t^n: mom5 of every cell (layer 0: moments_from_conserved(U);
// kinetic: moments_of(f) from the compact batch), L1 distances of the kinetic cells.
__global__ void view_kernel(int64_t cells, const int8_t* __restrict__ r, const double* __restrict__ U, double hr,
                            const int* __restrict__ pos, const double* __restrict__ momk,
                            const double* __restrict__ l1k, const int* __restrict__ stk, double* __restrict__ mom,
                            double* __restrict__ l1, HybCounts* cnt) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cells) return;
    double* m = mom + 5 * c;
    if (r[c] == 0) {
        if (!mom_from_u(U + 4 * c, hr, m)) {
            fail_at(cnt, c, HK_POSITIVITY);
            for (int e = 0; e < 5; ++e) m[e] = 1.0;  // keeps the classifier finite; the step fails
        }
        l1[c] = 0.0;
    } else {
        const int k = pos[c];
        for (int e = 0; e < 5; ++e) m[e] = momk[5 * k + e];
        l1[c] = l1k[k];
        if (stk[k]) {
            fail_at(cnt, c, stk[k]);
            m[0] = m[4] = 1.0;
        }
    }
}

// convert_on_transition (src/regime.cpp:54-72) 1 -> 0, the hydro view W fed to
// the Euler step, transition counts.
__global__ void convert_kernel(int64_t cells, const int8_t* __restrict__ r_old, const int8_t* __restrict__ r_new,
                               double* __restrict__ U, const double* __restrict__ mom, double hr,
                               double* __restrict__ W, HybCounts* cnt) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cells) return;
    const int ro = r_old[c], rn = r_new[c];
    double* w = W + 4 * c;
    if (ro == 0) {
        for (int e = 0; e < 4; ++e) w[e] = U[4 * c + e];
        if (rn != 0) atomicAdd(&cnt->n01, 1);
    } else {
        u_from_mom(mom + 5 * c, hr, w);
        if (rn == 0) {
            for (int e = 0; e < 4; ++e) U[4 * c + e] = w[e];
            atomicAdd(&cnt->n10, 1);
        }
    }
    if (rn == 0) atomicAdd(&cnt->n0, 1);
}

__device__ __forceinline__ bool kin_at(const int8_t* r, int nx, int ny, int i, int j) {
    i = (i % nx + nx) % nx;
    j = (j % ny + ny) % ny;
    return r[(int64_t)j * nx + i] != 0;
}

// Pass B (after the update): batch [K1 | K2] in cell order with their Knudsen
// numbers, and the Maxwellian targets: 0 -> 1 transitions and the layer-0
// cells on the periodic +-2 transport stencil of a kinetic cell, with the
// moments of their (post-conversion) hydro state.
__global__ void __launch_bounds__(kLT) list_new_kernel(int nx, int ny, const int8_t* __restrict__ r_old,
                                                       const int8_t* __restrict__ r_new,
                                                       const double* __restrict__ U, double hr,
                                                       const double* __restrict__ eps, int64_t* __restrict__ list,
                                                       int64_t* __restrict__ tmp2, double* __restrict__ eps_k,
                                                       int64_t* __restrict__ mlist, double* __restrict__ mmom,
                                                       HybCounts* cnt, int gx, int64_t* __restrict__ tmp2b,
                                                       int64_t* __restrict__ tmp2c) {
    __shared__ int wt[64];
    __shared__ int b1, b2, bm, b2b, b2c;
    const int64_t cells = (int64_t)nx * ny;
    if (threadIdx.x == 0) b1 = b2 = bm = b2b = b2c = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < cells; c0 += kLT) {
        const int64_t c = c0 + threadIdx.x;
        int rn = 0, ro = 0;
        bool halo = false;
        if (c < cells) {
            rn = r_new[c];
            ro = r_old[c];
            if (rn == 0) {
                const int i = int(c % nx), j = int(c / nx);
                for (int d = 1; d <= 2 && !halo; ++d)
                    halo = kin_at(r_new, nx, ny, i - d, j) || kin_at(r_new, nx, ny, i + d, j) ||
                           kin_at(r_new, nx, ny, i, j - d) || kin_at(r_new, nx, ny, i, j + d);
            }
        }
        const int gd = c < cells ? ghost_dist(int(c % nx), nx, gx) : 0;
        const int cls = gd == 0 ? 0 : (gd <= 2 ? 1 : 2);
        const int s1 = block_slot(rn == 1, wt, &b1);
        const int s2 = block_slot(rn == 2 && cls == 0, wt, &b2);
        const int s2b = block_slot(rn == 2 && cls == 1, wt, &b2b);
        const int s2c = block_slot(rn == 2 && cls == 2, wt, &b2c);
        const bool mw = halo || (ro == 0 && rn != 0);
        const int sm = block_slot(mw, wt, &bm);
        if (rn == 1) list[s1] = c;
        if (rn == 2) (cls == 0 ? tmp2[s2] : (cls == 1 ? tmp2b[s2b] : tmp2c[s2c])) = c;
        if (mw) {
            mlist[sm] = c;
            if (!mom_from_u(U + 4 * c, hr, mmom + 5 * sm)) {
                fail_at(cnt, c, HK_POSITIVITY);
                for (int e = 0; e < 5; ++e) mmom[5 * sm + e] = 1.0;
            }
        }
    }
    __syncthreads();
    const int n1 = b1, n2a = b2, n2b = b2b, n2c = b2c, n2 = n2a + n2b + n2c;
    for (int k = threadIdx.x; k < n2a; k += kLT) list[n1 + k] = tmp2[k];
    for (int k = threadIdx.x; k < n2b; k += kLT) list[n1 + n2a + k] = tmp2b[k];
    for (int k = threadIdx.x; k < n2c; k += kLT) list[n1 + n2a + n2b + k] = tmp2c[k];
    __syncthreads();
    for (int k = threadIdx.x; k < n1 + n2; k += kLT) eps_k[k] = eps[list[k]];
    if (threadIdx.x == 0) {
        cnt->n1 = n1;
        cnt->n2 = n2;
        cnt->n2a = n2a;
        cnt->n2b = n2b;
        cnt->nm = bm;
    }
}

// Layer-0 cells take the Euler result; the layer map advances.
__global__ void commit_kernel(int64_t cells, const int8_t* __restrict__ r_new, int8_t* __restrict__ r,
                              const double* __restrict__ W, double* __restrict__ U, int euler) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cells) return;
    const int rn = r_new[c];
    if (euler && rn == 0)
        for (int e = 0; e < 4; ++e) U[4 * c + e] = W[4 * c + e];
    r[c] = (int8_t)rn;
}

// Per-cell statuses of the batch (stage info: status | fallback << 8; residual status).
__global__ void status_kernel(int64_t nk, const int64_t* __restrict__ list, const int* __restrict__ st,
                              HybCounts* cnt, int nx, int gx) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nk) return;
    if (ghost_dist(int(list[k] % nx), nx, gx)) return;  // ghost results are discarded (their owner checks them)
    const int s = st[k] & 0xff;
    if (s && s != HK_NUMERICAL_CONSISTENCY) fail_at(cnt, list[k], s);
}

// pos[list[b]] = b for the batch rows (pos preset to -1)
__global__ void inverse_list_kernel(int64_t nk, const int64_t* __restrict__ list, int* __restrict__ pos) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b < nk) pos[list[b]] = int(b);
}

unsigned nblk(int64_t n, int t) { return unsigned((n + t - 1) / t); }

// Grow-only device buffer owned by the context.
int grow(hk_ctx ctx, void** p, size_t* have, size_t need, const char* what, size_t cap) {
    if (need <= *have) return HK_OK;
    if (*p) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(*p);
        *p = nullptr;
        *have = 0;
    }
    need = std::max(need, std::min(cap, need + need / 4));  // headroom: the kinetic batch grows step by step
    if (cudaMalloc(p, need) != cudaSuccess) return fail(ctx, HK_CUDA, std::string("hybrid step: cannot allocate ") + what);
    *have = need;
    return HK_OK;
}

template <class T>
T* carve(char*& p, int64_t count) {
    T* out = reinterpret_cast<T*>(p);
    p += (sizeof(T) * count + 255) & ~size_t(255);
    return out;
}

struct PR {
    double a_ex10, a_im00, a_im10, a_im11;
};
PR pr222_t() {  // ImexTableau::pr222 (inc/imex.hpp:23-34)
    const double C = 1.0 / std::sqrt(2.0);
    const double delta = 1.0 - 1.0 / (2.0 * C);
    return {1.0, 1.0 - C, C - delta, delta};
}

// HK_HYB_PROF=1 (profiling builds, -DHK_PROFILING=1): per-phase wall time (stream synchronised at each mark), stderr.
struct PhaseProf {
    bool on;
    cudaStream_t s;
    std::chrono::steady_clock::time_point t;
    std::string line;
    explicit PhaseProf(cudaStream_t st) : on(HK_PROFILING && getenv("HK_HYB_PROF") != nullptr), s(st) {
        if (on) {
            cudaStreamSynchronize(s);
            t = std::chrono::steady_clock::now();
        }
    }
    void mark(const char* name) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        char buf[64];
        snprintf(buf, sizeof buf, " %s %.2f", name, std::chrono::duration<double, std::milli>(now - t).count());
        line += buf;
        t = now;
    }
    ~PhaseProf() {
        if (on) fprintf(stderr, "[hk hybrid prof ms]%s\n", line.c_str());
    }
};

int read_counts(hk_ctx ctx, const HybCounts* dev, HybCounts& h, const char* what) {
    int st = check_cuda(ctx, cudaMemcpyAsync(&h, dev, sizeof h, cudaMemcpyDeviceToHost, ctx->stream), what);
    if (!st) st = check_cuda(ctx, cudaStreamSynchronize(ctx->stream), what);
    if (!st && h.bad != ~0ull)
        st = fail(ctx, int(h.bad & 0xff), std::string(what) + ": cell failed", int64_t(h.bad >> 8));
    return st;
}

}  // namespace
}  // namespace hk

using namespace hk;

extern "C" int hk_hybrid_step(hk_ctx ctx, hk_kernel k, int nx, int ny, double dx, double dy, double dt,
                              const double* eps_dev, int8_t* r_dev, double* hydro_dev, double* f_dev,
                              const hk_hybrid_params* p, int64_t* counts) {
    HK_RANGE("hk_hybrid_step");
    if (!ctx || !k || !p) return HK_CONTRACT;
    if (nx < 1 || ny < 1) return fail(ctx, HK_CONTRACT, "hybrid step: empty grid");
    // every argument check precedes the first launch: a rejected call leaves the state untouched
    if (p->ghost_x < 0 || 2 * p->ghost_x >= nx)
        return fail(ctx, HK_CONTRACT, "hybrid step: ghost_x must be in [0, nx / 2)");
    if (p->update_regimes && (!(p->eta0 > 0.0) || !(p->eta1 > 0.0) || !(p->delta0 > 0.0)))
        return fail(ctx, HK_CONFIG, "regime thresholds eta0, eta1, delta0 must be positive");
    cudaSetDevice(ctx->device);
    ctx->err_cell = -1;
    const int n = k->n;
    const double vmax = k->vmax, hr = p->heat_ratio;
    const int64_t cells = (int64_t)nx * ny, nb = (int64_t)n * n * n;
    cudaStream_t s = ctx->stream;
    int st;
    PhaseProf prof(s);

    // ---- per-cell workspace (fixed per grid) ----
    const size_t small_need = 256 * 16 + (sizeof(double) * cells * (5 + 1 + 4 + 8 + 5 + 5 + 1 + 1) +
                                          sizeof(int64_t) * cells * 6 + sizeof(int) * cells * 3 + cells * 2 + 4096);
    if ((st = grow(ctx, &ctx->hyb_small, &ctx->hyb_small_bytes, small_need, "per-cell workspace", small_need)))
        return st;
    char* q = static_cast<char*>(ctx->hyb_small);
    HybCounts* cnt = carve<HybCounts>(q, 1);
    double* mom = carve<double>(q, 5 * cells);
    double* l1 = carve<double>(q, cells);
    double* W = carve<double>(q, 4 * cells);
    double* ework = carve<double>(q, 8 * cells);
    double* momk = carve<double>(q, 5 * cells);
    double* mmom = carve<double>(q, 5 * cells);
    double* l1k = carve<double>(q, cells);
    double* eps_k = carve<double>(q, cells);
    int64_t* list = carve<int64_t>(q, cells);
    int64_t* tmp2 = carve<int64_t>(q, cells);
    int64_t* mlist = carve<int64_t>(q, cells);
    int64_t* list_old = carve<int64_t>(q, cells);
    int64_t* tmp2b = carve<int64_t>(q, cells);
    int64_t* tmp2c = carve<int64_t>(q, cells);
    int* pos = carve<int>(q, cells);
    int* stk = carve<int>(q, cells);
    int* stk2 = carve<int>(q, cells);
    int8_t* r_new = carve<int8_t>(q, cells);

    HybCounts h0{};
    h0.bad = ~0ull;
    cudaMemcpyAsync(cnt, &h0, sizeof h0, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(stk, 0, sizeof(int) * cells, s);

    // ---- 1. indicator pass at t^n ----
    list_old_kernel<<<1, kLT, 0, s>>>(cells, r_dev, list_old, pos, cnt);
    if ((st = moments_launch(ctx, n, vmax, f_dev, cells, momk, nullptr, nullptr, l1k, stk, list_old, &cnt->nk_old)))
        return st;
    view_kernel<<<nblk(cells, 128), 128, 0, s>>>(cells, r_dev, hydro_dev, hr, pos, momk, l1k, stk, mom, l1, cnt);
    ctx->launches += 2;
    if (p->update_regimes) {
        ClassifyParams cp{nx, ny, dx, dy, p->mu0, p->kappa0, p->eta0, p->eta1, p->delta0, p->signed_sum};
        if ((st = classify_launch(ctx, cp, mom, eps_dev, l1, r_dev, r_new, nullptr, nullptr))) return st;
    } else {
        cudaMemcpyAsync(r_new, r_dev, cells, cudaMemcpyDeviceToDevice, s);
    }
    // ---- 2. conversion + the lists of the step ----
    convert_kernel<<<nblk(cells, 128), 128, 0, s>>>(cells, r_dev, r_new, hydro_dev, mom, hr, W, cnt);
    const int gx = p->ghost_x;
    list_new_kernel<<<1, kLT, 0, s>>>(nx, ny, r_dev, r_new, hydro_dev, hr, eps_dev, list, tmp2, eps_k, mlist, mmom, cnt,
                                      gx, tmp2b, tmp2c);
    ctx->launches += 2;
    if ((st = check_cuda(ctx, cudaGetLastError(), "hybrid lists"))) return st;
    HybCounts h{};
    if ((st = read_counts(ctx, cnt, h, "hybrid_step indicator pass"))) return st;
    const int64_t n1 = h.n1, n2 = h.n2, nk = n1 + n2, nm = h.nm;
    // layer-2 cells whose residual is needed: at Y1 classes A + B, at Y2 class A (all of K2 on a plain torus)
    const int64_t n2_y1 = h.n2a + h.n2b, n2_y2 = h.n2a;
    prof.mark("indicators");
    // Maxwellians of the 0 -> 1 cells and of the layer-0 transport halo
    if (nm && (st = maxwellian_launch(ctx, n, vmax, mmom, nm, f_dev, nullptr, mlist, nullptr))) return st;
    prof.mark("halo");

    // ---- 3. layer 0: TVD-RK2 of the hydro view ----
    const bool euler = h.n0 > 0;
    if (euler && (st = hk_euler_tvd_rk2_step(ctx, W, nx, ny, dx, dy, dt, hr, p->eps_weno, ework))) return st;
    prof.mark("euler");

    // ---- 4. kinetic layers: PR(2,2,2) on the compact batch ----
    if (nk) {
        TransportParams tp{n, vmax, nx, ny, 0, dx, dy, p->eps_weno};
        // the lane sweep writes T straight into the batch rows (pos: cell -> batch row);
        // otherwise a dense T field is gathered
        const bool compact_T = transport_lanes_path(tp);
        const int64_t t_cells = compact_T ? 0 : cells;
        const size_t big_need = sizeof(double) * (size_t)nb * (size_t)(7 * nk + t_cells) + 8 * 256;
        const size_t big_max = sizeof(double) * (size_t)nb * (size_t)(7 * cells + t_cells) + 8 * 256;  // all kinetic
        if ((st = grow(ctx, &ctx->hyb_big, &ctx->hyb_big_bytes, big_need, "kinetic workspace", big_max))) return st;
        char* b = static_cast<char*>(ctx->hyb_big);
        double* fk = carve<double>(b, nk * nb);
        double* Y = carve<double>(b, nk * nb);
        double* k1 = carve<double>(b, nk * nb);
        double* q1 = carve<double>(b, nk * nb);
        double* tr = carve<double>(b, nk * nb);
        double* res = carve<double>(b, nk * nb);
        double* fa = carve<double>(b, nk * nb);
        double* T = compact_T ? nullptr : carve<double>(b, cells * nb);
        if (compact_T) {  // pos (free since the indicator pass) becomes the inverse of list
            cudaMemsetAsync(pos, 0xff, sizeof(int) * cells, s);
            inverse_list_kernel<<<nblk(nk, 256), 256, 0, s>>>(nk, list, pos);
            ctx->launches++;
            tp.out_pos = pos;
        }
        const PR t = pr222_t();
        cudaMemsetAsync(stk, 0, sizeof(int) * nk, s);
        cudaMemsetAsync(stk2, 0, sizeof(int) * nk, s);
        uint8_t* act = reinterpret_cast<uint8_t*>(ework);  // the Euler work is free again
        if ((st = transport_row_activity(ctx, nx, ny, r_new, act))) return st;
        tp.row_act = act;  // T is only gathered at the kinetic cells
        auto stages = [&](const double* fin, double a, double* out, double* k1o) -> int {
            int e = HK_OK;
            if (n1)
                e = stage_launch(ctx, true, n, vmax, fin, out, n1, a, eps_k, 0.0, p->esbgk_beta, p->nu_coeff, stk,
                                 nullptr, k1o, 1.0 / t.a_im00);
            if (!e && n2)
                e = stage_launch(ctx, false, n, vmax, fin + n1 * nb, out + n1 * nb, n2, a, eps_k + n1, 0.0, 0.0,
                                 p->pen_coeff, stk + n1, nullptr, k1o ? k1o + n1 * nb : nullptr, 1.0 / t.a_im00);
            return e;
        };
        auto residual = [&](const double* y, int64_t m2) -> int {  // penalized_residual of the first m2 layer-2 cells
            if (p->residual_fn) {
                const int e = p->residual_fn(p->residual_user, m2 ? y + n1 * nb : nullptr, m2 ? res + n1 * nb : nullptr,
                                             m2, m2 ? stk2 + n1 : nullptr, (void*)s);
                return e ? fail(ctx, e, "hybrid step: residual hook failed") : HK_OK;
            }
            if (!m2) return HK_OK;
            int e = collision_launch(ctx, k, y + n1 * nb, res + n1 * nb, m2, p->coll_flags & ~HK_COLL_STRICT, nullptr);
            return e ? e : residual_finish_launch(ctx, n, vmax, y + n1 * nb, res + n1 * nb, m2, p->pen_coeff, stk2 + n1);
        };
        auto transport = [&](const double* y) -> int {  // T(y) at the batch cells
            if (compact_T) {  // the sweep reads y from the batch rows and writes T to them: no copies
                TransportParams ty = tp;
                ty.in_pos = pos;
                ty.in_batch = y;
                return transport_launch(ctx, ty, f_dev, tr);
            }
            int e = hk_scatter_cells(ctx, nb, y, list, nk, f_dev);
            if (!e) e = transport_launch(ctx, tp, f_dev, T);
            if (!e) e = hk_gather_cells(ctx, nb, T, list, nk, tr);
            return e;
        };
        // q = tr (+ res / eps on the layer-2 part), via the IMEX combinations
        // batch ranges [b0, b1) with (with_res) or without the residual term
        auto explicit_part = [&](int op, double* o, const double* y, int64_t m2) -> int {
            auto range = [&](int64_t b0, int64_t b1, bool with_res) -> int {
                if (b1 <= b0) return HK_OK;
                return combine_launch(ctx, op, (b1 - b0) * nb, nb, dt, eps_k + b0, o + b0 * nb, nullptr,
                                      y ? y + b0 * nb : nullptr, q1 + b0 * nb, k1 + b0 * nb, tr + b0 * nb,
                                      with_res ? res + b0 * nb : nullptr);
            };
            int e = range(0, n1, false);
            if (!e) e = range(n1, n1 + m2, true);
            if (!e) e = range(n1 + m2, nk, false);  // ghost cells whose result is not needed
            return e;
        };
        st = hk_gather_cells(ctx, nb, f_dev, list, nk, fk);                               // f^n of the batch
        prof.mark("gather");
        auto check_status = [&](const int* arr) {  // statuses are overwritten by the next phase: fold them now
            status_kernel<<<nblk(nk, 256), 256, 0, s>>>(nk, list, arr, cnt, nx, gx);
            ctx->launches++;
        };
        if (!st) st = stages(fk, t.a_im00 * dt, Y, k1);                                   // Y1, k1
        if (!st) check_status(stk);
        prof.mark("stage1");
        if (!st) st = transport(Y);                                                       // T(Y1)
        prof.mark("transport1");
        if (!st) st = residual(Y, n2_y1);                                                 // res(Y1)
        if (!st) check_status(stk2);
        prof.mark("residual1");
        if (!st) st = explicit_part(1, q1, nullptr, n2_y1);                               // q1
        prof.mark("combine");
        if (stage_acc_supported(n)) {  // Y2 = stage(f + dt a_ex10 q1 + a_im10 k1), f_acc formed in the stage
            const double cq = dt * t.a_ex10, ck = t.a_im10;
            if (!st && n1)
                st = stage_acc_launch(ctx, true, n, vmax, fk, q1, k1, cq, ck, Y, n1, t.a_im11 * dt, eps_k, p->esbgk_beta,
                                      p->nu_coeff, stk);
            if (!st && n2)
                st = stage_acc_launch(ctx, false, n, vmax, fk + n1 * nb, q1 + n1 * nb, k1 + n1 * nb, cq, ck, Y + n1 * nb,
                                      n2, t.a_im11 * dt, eps_k + n1, 0.0, p->pen_coeff, stk + n1);
        } else {
            if (!st) st = combine_launch(ctx, 2, nk * nb, nb, dt, eps_k, fa, fk, nullptr, q1, k1, nullptr, nullptr);
            if (!st) st = stages(fa, t.a_im11 * dt, Y, nullptr);                          // Y2
        }
        prof.mark("stage2");
        if (!st) st = transport(Y);                                                       // T(Y2)
        prof.mark("transport2");
        if (!st) st = residual(Y, n2_y2);                                                 // res(Y2)
        prof.mark("residual2");
        if (!st) st = explicit_part(3, fk, Y, n2_y2);                                     // final, in place
        if (!st) st = hk_scatter_cells(ctx, nb, fk, list, nk, f_dev);
        prof.mark("final");
        if (!st) {
            check_status(stk);   // stage 2
            check_status(stk2);  // residual at Y2 (cells past n1 + n2_y2 keep their Y1 status: ghosts, skipped)
        }
        if (st) return st;
    } else if (p->residual_fn) {  // no kinetic cell here: still take part in both (collective) hook calls
        for (int k2 = 0; k2 < 2; ++k2)
            if ((st = p->residual_fn(p->residual_user, nullptr, nullptr, 0, nullptr, (void*)s)))
                return fail(ctx, st, "hybrid step: residual hook failed");
    }
    commit_kernel<<<nblk(cells, 256), 256, 0, s>>>(cells, r_new, r_dev, W, hydro_dev, euler ? 1 : 0);
    ctx->launches++;
    if ((st = check_cuda(ctx, cudaGetLastError(), "hybrid commit"))) return st;
    HybCounts e{};
    if ((st = read_counts(ctx, cnt, e, "hybrid_step stage updates"))) return st;
    if (counts) {
        counts[0] = e.n0;
        counts[1] = e.n1;
        counts[2] = e.n2;
        counts[3] = e.n01;
        counts[4] = e.n10;
        counts[5] = e.nm - e.n01;
    }
    return HK_OK;
}

// ---------------------------------------------------------------------------
// hk_hybrid_step on one x-slab, host logic in C++ (the C-ABI twin of
// partition.hybrid_step_slab): one exchange of `ghost` columns of (r, eps,
// hydro, f) per side straight into a padded [ny][nx_local + 2 ghost] copy of
// the slab (NCCL send/recv on the context communicator, or the slab's own wrap
// without one), the step on the padded local torus with ghost_x = ghost (ghost
// cells get only the residuals an interior cell depends on), the interior
// copied back, and the layer counts of the interior all-reduced over the
// communicator.  With ghost >= the step's x-dependency radius (7 cells;
// partition.HYB_GHOST = 8) the interior equals the global step's.
// ---------------------------------------------------------------------------
namespace hk {
namespace {
__global__ void layer_count_kernel(int64_t cells, const int8_t* __restrict__ r, double* __restrict__ out) {
    __shared__ unsigned c[3];
    if (threadIdx.x < 3) c[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cells; i += (int64_t)gridDim.x * blockDim.x) {
        const int v = r[i];
        if (v >= 0 && v <= 2) atomicAdd(&c[v], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 3 && c[threadIdx.x]) atomicAdd(out + threadIdx.x, double(c[threadIdx.x]));
}
}  // namespace
}  // namespace hk

extern "C" int hk_hybrid_step_slab(hk_ctx ctx, hk_kernel k, int nx_local, int ny, double dx, double dy, double dt,
                                   const double* eps_dev, int8_t* r_dev, double* hydro_dev, double* f_dev,
                                   const hk_hybrid_params* p, int ghost, int64_t* counts) {
    HK_RANGE("hk_hybrid_step_slab");
    if (!ctx || !k || !p) return HK_CONTRACT;
    if (ghost < 1 || nx_local < ghost || ny < 1)
        return fail(ctx, HK_CONTRACT, "hybrid slab step: need 1 <= ghost <= nx_local and ny >= 1");
    cudaSetDevice(ctx->device);
    const int w = ghost, nxp = nx_local + 2 * w;
    const int64_t nb = (int64_t)k->n * k->n * k->n, cells = (int64_t)nx_local * ny, cp = (int64_t)nxp * ny;
    // padded workspace: [counts 3][r cp][eps cp][hydro 4 cp][f nb cp], 256-byte aligned pieces
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t need = al(3 * sizeof(double)) + al(cp) + al(sizeof(double) * cp) + al(sizeof(double) * 4 * cp) +
                        al(sizeof(double) * (size_t)nb * cp);
    int st;
    if ((st = grow(ctx, &ctx->slab_pad, &ctx->slab_pad_bytes, need, "padded slab", need))) return st;
    char* q = static_cast<char*>(ctx->slab_pad);
    double* cnt = carve<double>(q, 3);
    int8_t* r_p = carve<int8_t>(q, cp);
    double* e_p = carve<double>(q, cp);
    double* h_p = carve<double>(q, 4 * cp);
    double* f_p = carve<double>(q, nb * cp);
    struct Field {
        const void* src;
        void* pad;
        size_t cb;
    };
    const Field fields[4] = {{r_dev, r_p, 1}, {eps_dev, e_p, sizeof(double)}, {hydro_dev, h_p, 4 * sizeof(double)},
                             {f_dev, f_p, sizeof(double) * (size_t)nb}};
    cudaStream_t s = ctx->stream;
    for (const Field& fl : fields) {  // interior, then the ghost columns
        const size_t row = fl.cb * nx_local, prow = fl.cb * nxp;
        if ((st = check_cuda(ctx, cudaMemcpy2DAsync(static_cast<char*>(fl.pad) + fl.cb * w, prow, fl.src, row, row, ny,
                                                    cudaMemcpyDeviceToDevice, s), "slab padding")))
            return st;
        if ((st = halo_columns_padded(ctx, fl.src, fl.cb, nx_local, ny, w, fl.pad))) return st;
    }
    hk_hybrid_params q2 = *p;
    q2.ghost_x = w;
    if ((st = hk_hybrid_step(ctx, k, nxp, ny, dx, dy, dt, e_p, r_p, h_p, f_p, &q2, nullptr))) return st;
    const Field back[3] = {{r_p, r_dev, 1}, {h_p, hydro_dev, 4 * sizeof(double)}, {f_p, f_dev, sizeof(double) * (size_t)nb}};
    for (const Field& fl : back) {
        const size_t row = fl.cb * nx_local, prow = fl.cb * nxp;
        if ((st = check_cuda(ctx, cudaMemcpy2DAsync(fl.pad, row, static_cast<const char*>(fl.src) + fl.cb * w, prow, row, ny,
                                                    cudaMemcpyDeviceToDevice, s), "slab unpadding")))
            return st;
    }
    // layer counts of the interior, summed over the ranks
    cudaMemsetAsync(cnt, 0, 3 * sizeof(double), s);
    layer_count_kernel<<<unsigned(std::min<int64_t>((cells + 255) / 256, 4LL * ctx->sm_count)), 256, 0, s>>>(cells, r_dev, cnt);
    ctx->launches++;
    if ((st = check_cuda(ctx, cudaGetLastError(), "layer counts"))) return st;
    if (ctx->comm && ctx->nranks > 1 && (st = hk_allreduce_scalars(ctx, cnt, 3, HK_REDUCE_SUM))) return st;
    double h[3];
    if ((st = check_cuda(ctx, cudaMemcpyAsync(h, cnt, sizeof h, cudaMemcpyDeviceToHost, s), "counts D2H")) ||
        (st = check_cuda(ctx, cudaStreamSynchronize(s), "counts sync")))
        return st;
    if (counts)
        for (int i = 0; i < 3; ++i) counts[i] = (int64_t)h[i];
    return HK_OK;
}
