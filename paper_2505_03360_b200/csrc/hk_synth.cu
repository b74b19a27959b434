// hk_synth.cu — cross-layer stencil synthesis on the device (SURVEY §8f "next" #1).
//
//   synthesize_hydro_state    src/coupling.cpp:57-70
//   synthesize_distribution   src/coupling.cpp:72-93
//   SpatialGrid::clamp_interior  src/grid.cpp:12-16
//
// What a stencil at cell (i, j) sees, per the reference: ghost cells read the
// closest interior cell; obstacle cells the fixed state (or its Maxwellian);
// layer-0 cells their conserved state (or its Maxwellian); kinetic cells their
// moments (or their stored block, verbatim).  The reference evaluates this
// per stencil access; here one call resolves a whole field (hydro) or a list
// of cells (distributions), in three stream-ordered kernels and one final
// 16-byte read-back:
//   1. resolve: one thread per target cell picks the source cell and the case,
//      writes the trivial cases directly and appends the rest to compact
//      device lists (Maxwellians: moments; copies: source cell; moments_of:
//      source cell), recording the lowest failing target by atomicMin;
//   2. the per-cell workers (maxwellian_kernel / moments kernels / a block
//      copy) consume the lists, their lengths read on the device;
//   3. (hydro) the moments are turned into conserved states.
// Compiled without FMA contraction (the conserved-state arithmetic is the
// reference's, bitwise).
#include <algorithm>
#include <cstdint>
#include <string>

#include "hk_cells.cuh"
#include "hk_internal.h"

namespace hk {
namespace {

constexpr int kGhost = 4;  // SpatialGrid::ghost_depth
constexpr int kStencil = 2;  // transport stencil half-width (src/transport.cpp:25-49)

struct Grid2 {
    int nx, ny;
    __device__ bool ghost(int i, int j) const { return i < kGhost || i >= nx - kGhost || j < kGhost || j >= ny - kGhost; }
    __device__ int64_t clamp(int i, int j) const {
        if (ghost(i, j)) {
            const int ilo = kGhost, ihi = nx - kGhost - 1, jlo = kGhost, jhi = ny - kGhost - 1;
            i = i < ilo ? ilo : (i > ihi ? ihi : i);
            j = j < jlo ? jlo : (j > jhi ? jhi : j);
        }
        return (int64_t)j * nx + i;
    }
};

struct FixedState {
    double u[4], mom[5];
    bool ok;  // maxwellian(obstacle_moments) does not throw
};

struct Lists {
    unsigned long long bad;  // (target << 8) | status, lowest first
    int n_maxw, n_copy, n_mom, pad;
};

__device__ void fail_at(Lists* l, int64_t key, int code) {
    atomicMin(&l->bad, ((unsigned long long)key << 8) | (unsigned)code);
}

// A cell is "kinetic" for the stencil when it is integrated by a kinetic layer.
__device__ bool kinetic_cell(const Grid2& g, const int8_t* r, const uint8_t* kind, int i, int j) {
    const int64_t c = (int64_t)j * g.nx + i;
    return !g.ghost(i, j) && kind[c] != HK_CELL_OBSTACLE && r[c] != 0;
}

// Distribution targets.  list mode (idx != null): target k is cell idx[k], its
// block goes to out[k]; stencil mode: every cell that is not kinetic but lies
// on the cross-shaped transport stencil of a kinetic cell, block in place.
__global__ void synth_dist_resolve_kernel(Grid2 g, const int8_t* __restrict__ r, const uint8_t* __restrict__ kind,
                                          const double* __restrict__ hydro, double hr, FixedState fx,
                                          const int64_t* __restrict__ idx, int64_t count, Lists* __restrict__ l,
                                          int64_t* __restrict__ maxw_dst, double* __restrict__ maxw_mom,
                                          int64_t* __restrict__ copy_dst, int64_t* __restrict__ copy_src) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    const int64_t cell = idx ? idx[k] : k;
    const int i = int(cell % g.nx), j = int(cell / g.nx);
    if (!idx) {
        if (kinetic_cell(g, r, kind, i, j)) return;
        bool read = false;
        for (int d = -kStencil; d <= kStencil && !read; ++d) {
            if (d == 0) continue;
            if (i + d >= 0 && i + d < g.nx) read = kinetic_cell(g, r, kind, i + d, j);
            if (!read && j + d >= 0 && j + d < g.ny) read = kinetic_cell(g, r, kind, i, j + d);
        }
        if (!read) return;
    }
    const int64_t tgt = idx ? k : cell;
    const int64_t src = g.clamp(i, j);
    if (kind[src] == HK_CELL_OBSTACLE) {
        if (!fx.ok) return fail_at(l, k, HK_DEGENERATE);
        const int q = atomicAdd(&l->n_maxw, 1);
        maxw_dst[q] = tgt;
        for (int e = 0; e < 5; ++e) maxw_mom[5 * q + e] = fx.mom[e];
    } else if (r[src] == 0) {  // maxwellian(moments_from_conserved(hydro)); pressure() throws first
        const double* u = hydro + 4 * src;
        if (!(u[0] > 0.0)) return fail_at(l, k, HK_POSITIVITY);
        const double p = (hr - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
        if (!(p > 0.0)) return fail_at(l, k, HK_POSITIVITY);
        if (!(p / u[0] > 0.0)) return fail_at(l, k, HK_DEGENERATE);
        const int q = atomicAdd(&l->n_maxw, 1);
        maxw_dst[q] = tgt;
        maxw_mom[5 * q + 0] = u[0];
        maxw_mom[5 * q + 1] = u[1] / u[0];
        maxw_mom[5 * q + 2] = u[2] / u[0];
        maxw_mom[5 * q + 3] = 0.0;
        maxw_mom[5 * q + 4] = p / u[0];
    } else if (idx || src != cell) {  // the stored block, verbatim
        const int q = atomicAdd(&l->n_copy, 1);
        copy_dst[q] = tgt;
        copy_src[q] = src;
    }
}

// On a failure nothing is written (the lists are emptied before the workers run).
__global__ void synth_gate_kernel(Lists* l) {
    if (l->bad != ~0ull) l->n_maxw = l->n_copy = l->n_mom = 0;
}

__global__ void block_copy_kernel(int64_t nb, const int* __restrict__ count_dev, const int64_t* __restrict__ dst_idx,
                                  const int64_t* __restrict__ src_idx, const double* __restrict__ src,
                                  double* __restrict__ dst) {
    const int64_t count = *count_dev;
    for (int64_t k = blockIdx.y; k < count; k += gridDim.y) {
        const double* sp = src + src_idx[k] * nb;
        double* dp = dst + dst_idx[k] * nb;
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nb; e += (int64_t)gridDim.x * blockDim.x)
            dp[e] = sp[e];
    }
}

// Hydro targets: every cell of the grid.
__global__ void synth_hydro_resolve_kernel(Grid2 g, const int8_t* __restrict__ r, const uint8_t* __restrict__ kind,
                                           const double* __restrict__ hydro, FixedState fx, Lists* __restrict__ l,
                                           int64_t* __restrict__ mom_dst, int64_t* __restrict__ mom_src,
                                           double* __restrict__ out) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= (int64_t)g.nx * g.ny) return;
    const int64_t src = g.clamp(int(c % g.nx), int(c / g.nx));
    if (kind[src] == HK_CELL_OBSTACLE) {
        for (int e = 0; e < 4; ++e) out[4 * c + e] = fx.u[e];
    } else if (r[src] == 0) {
        for (int e = 0; e < 4; ++e) out[4 * c + e] = hydro[4 * src + e];
    } else {
        const int q = atomicAdd(&l->n_mom, 1);
        mom_dst[q] = c;
        mom_src[q] = src;
    }
}

// conserved_from_moments(moments_of(f)) (src/coupling.cpp:15-22)
__global__ void synth_hydro_finish_kernel(Lists* l, double hr,
                                          const int64_t* __restrict__ mom_dst, const double* __restrict__ mom,
                                          const int* __restrict__ status, double* __restrict__ out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= l->n_mom) return;
    const int64_t c = mom_dst[k];
    if (status[k]) return fail_at(l, c, status[k]);
    const double* m = mom + 5 * k;
    const double rho = m[0];
    const double u2 = m[1] * m[1] + m[2] * m[2] + m[3] * m[3];
    out[4 * c + 0] = rho;
    out[4 * c + 1] = rho * m[1];
    out[4 * c + 2] = rho * m[2];
    out[4 * c + 3] = rho * m[4] / (hr - 1.0) + 0.5 * rho * u2;
}

unsigned blocks_of(int64_t n) { return unsigned((n + 255) / 256); }

int check_args(hk_ctx ctx, int n, int64_t nx, int64_t ny, const char* what) {
    if (nx < 2 * kGhost + 1 || ny < 2 * kGhost + 1 || nx * ny > (int64_t(1) << 31))
        return fail(ctx, HK_CONFIG, std::string(what) + ": the 4-cell ghost frame leaves no interior");
    if (n < 2 || n > 128) return fail(ctx, HK_UNSUPPORTED, std::string(what) + ": 2 <= n <= 128");
    return HK_OK;
}

// obstacle_state / obstacle_moments (src/coupling.cpp:39-53), host arithmetic
FixedState fixed_of(const hk_obstacle_spec* s, double hr) {
    FixedState fx{};
    if (!s) return fx;
    const double T = s->pressure / s->rho;
    fx.mom[0] = s->rho;
    fx.mom[1] = s->ux;
    fx.mom[2] = s->uy;
    fx.mom[3] = 0.0;
    fx.mom[4] = T;
    fx.u[0] = s->rho;
    fx.u[1] = s->rho * s->ux;
    fx.u[2] = s->rho * s->uy;
    const double u2 = s->ux * s->ux + s->uy * s->uy + 0.0 * 0.0;
    fx.u[3] = s->rho * T / (hr - 1.0) + 0.5 * s->rho * u2;
    fx.ok = (s->rho > 0.0) && (T > 0.0);
    return fx;
}

int finish(hk_ctx ctx, Lists* l, void* w, const char* what, int64_t* filled, bool by_list) {
    Lists h;
    int st = check_cuda(ctx, cudaMemcpyAsync(&h, l, sizeof h, cudaMemcpyDeviceToHost, ctx->stream), what);
    if (!st) st = check_cuda(ctx, cudaStreamSynchronize(ctx->stream), what);
    cudaFreeAsync(w, ctx->stream);
    if (st) return st;
    if (h.bad != ~0ull) {
        const int code = int(h.bad & 0xff);
        return fail(ctx, code,
                    std::string(what) + (code == HK_POSITIVITY ? ": non-positive density or pressure"
                                                               : ": degenerate state (rho <= 0 or T <= 0)") +
                        (by_list ? " (list entry)" : " (cell)"),
                    (int64_t)(h.bad >> 8));
    }
    if (filled) *filled = int64_t(h.n_maxw) + h.n_copy;
    return HK_OK;
}

}  // namespace
}  // namespace hk

using namespace hk;

extern "C" {

int hk_synthesize_hydro(hk_ctx ctx, int n, double vmax, int64_t nx, int64_t ny, const hk_obstacle_spec* spec,
                        const int8_t* r_dev, const uint8_t* kind_dev, const double* hydro_dev, const double* f_dev,
                        double heat_ratio, double* out_dev) {
    int st = check_args(ctx, n, nx, ny, "synthesize_hydro_state");
    if (st) return st;
    cudaSetDevice(ctx->device);
    const int64_t cells = nx * ny;
    const size_t o_dst = 256, o_src = o_dst + 8 * cells, o_mom = o_src + 8 * cells, o_st = o_mom + 40 * cells,
                 bytes = o_st + 4 * cells;
    char* w = nullptr;
    if (cudaMallocAsync(&w, bytes, ctx->stream) != cudaSuccess) return fail(ctx, HK_CUDA, "synthesize alloc");
    Lists* l = reinterpret_cast<Lists*>(w);
    int64_t* mdst = reinterpret_cast<int64_t*>(w + o_dst);
    int64_t* msrc = reinterpret_cast<int64_t*>(w + o_src);
    double* mom = reinterpret_cast<double*>(w + o_mom);
    int* mst = reinterpret_cast<int*>(w + o_st);
    cudaMemsetAsync(l, 0xff, sizeof(unsigned long long), ctx->stream);
    cudaMemsetAsync(&l->n_maxw, 0, 4 * sizeof(int), ctx->stream);
    const Grid2 g{int(nx), int(ny)};
    synth_hydro_resolve_kernel<<<blocks_of(cells), 256, 0, ctx->stream>>>(g, r_dev, kind_dev, hydro_dev,
                                                                           fixed_of(spec, heat_ratio), l, mdst, msrc,
                                                                           out_dev);
    ctx->launches++;
    st = check_cuda(ctx, cudaGetLastError(), "synthesize hydro");
    if (!st) st = moments_launch(ctx, n, vmax, f_dev, cells, mom, nullptr, nullptr, nullptr, mst, msrc, &l->n_mom);
    if (!st) {
        synth_hydro_finish_kernel<<<blocks_of(cells), 256, 0, ctx->stream>>>(l, heat_ratio, mdst, mom, mst, out_dev);
        ctx->launches++;
        st = check_cuda(ctx, cudaGetLastError(), "synthesize hydro");
    }
    if (st) {
        cudaFreeAsync(w, ctx->stream);
        return st;
    }
    return finish(ctx, l, w, "synthesize_hydro_state", nullptr, false);
}

int hk_synthesize_distributions(hk_ctx ctx, int n, double vmax, int64_t nx, int64_t ny, const hk_obstacle_spec* spec,
                                const int8_t* r_dev, const uint8_t* kind_dev, const double* hydro_dev, double* f_dev,
                                double heat_ratio, const int64_t* idx_dev, int64_t count, double* out_dev,
                                int64_t* filled) {
    HK_RANGE("hk_synthesize_distributions");
    if (filled) *filled = 0;
    int st = check_args(ctx, n, nx, ny, "synthesize_distribution");
    if (st) return st;
    const bool list = idx_dev != nullptr;
    if (list && (count < 0 || (count > 0 && !out_dev)))
        return fail(ctx, HK_CONTRACT, "synthesize_distribution: list mode needs out_dev [count][n^3]");
    const int64_t cells = nx * ny, targets = list ? count : cells;
    if (targets == 0) return HK_OK;
    cudaSetDevice(ctx->device);
    const size_t o_md = 256, o_mm = o_md + 8 * targets, o_cd = o_mm + 40 * targets, o_cs = o_cd + 8 * targets,
                 bytes = o_cs + 8 * targets;
    char* w = nullptr;
    if (cudaMallocAsync(&w, bytes, ctx->stream) != cudaSuccess) return fail(ctx, HK_CUDA, "synthesize alloc");
    Lists* l = reinterpret_cast<Lists*>(w);
    int64_t* md = reinterpret_cast<int64_t*>(w + o_md);
    double* mm = reinterpret_cast<double*>(w + o_mm);
    int64_t* cd = reinterpret_cast<int64_t*>(w + o_cd);
    int64_t* cs = reinterpret_cast<int64_t*>(w + o_cs);
    cudaMemsetAsync(l, 0xff, sizeof(unsigned long long), ctx->stream);
    cudaMemsetAsync(&l->n_maxw, 0, 4 * sizeof(int), ctx->stream);
    const Grid2 g{int(nx), int(ny)};
    synth_dist_resolve_kernel<<<blocks_of(targets), 256, 0, ctx->stream>>>(
        g, r_dev, kind_dev, hydro_dev, heat_ratio, fixed_of(spec, heat_ratio), idx_dev, targets, l, md, mm, cd, cs);
    synth_gate_kernel<<<1, 1, 0, ctx->stream>>>(l);
    ctx->launches += 2;
    st = check_cuda(ctx, cudaGetLastError(), "synthesize distributions");
    double* dst = list ? out_dev : f_dev;
    if (!st) st = maxwellian_launch(ctx, n, vmax, mm, targets, dst, nullptr, md, &l->n_maxw);
    if (!st) {
        const int64_t nb = int64_t(n) * n * n;
        const dim3 grid(unsigned(std::min<int64_t>((nb + 255) / 256, 64)), unsigned(std::min<int64_t>(targets, 65535)));
        block_copy_kernel<<<grid, 256, 0, ctx->stream>>>(nb, &l->n_copy, cd, cs, f_dev, dst);
        ctx->launches++;
        st = check_cuda(ctx, cudaGetLastError(), "synthesize copies");
    }
    if (st) {
        cudaFreeAsync(w, ctx->stream);
        return st;
    }
    return finish(ctx, l, w, "synthesize_distribution", filled, list);
}

}  // extern "C"
