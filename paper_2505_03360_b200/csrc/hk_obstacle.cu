// hk_obstacle.cu — embedded obstacles on the device (SURVEY §8f "next" #4).
//
//   classify_cells        src/grid.cpp:74-110 (in_obstacle_footprint :56-72)
//   apply_obstacle        src/coupling.cpp:95-147 (obstacle_state / _moments :39-53)
//
// The reference walks the cells in row-major order and throws at the first
// failing one, leaving the earlier cells updated.  Here every cell is one
// thread: a first kernel classifies the moved footprint and finds, by an
// atomicMin over (cell << 8 | status), the cell the reference would throw at;
// a second applies the update to the cells before it (and the partial update
// the reference leaves on the failing cell itself) and appends the cells that
// need a Maxwellian block to a compact list; maxwellian_kernel then writes
// those blocks in place in the dense field.  Compiled without FMA contraction:
// r, kind and hydro are bitwise the reference's (tests/test_gpu_obstacle.py).
#include <cstdint>
#include <string>

#include "hk_cells.cuh"
#include "hk_internal.h"

namespace hk {
namespace {

constexpr int kGhost = 4;  // SpatialGrid::ghost_depth
constexpr int kRing = 2;   // forced-kinetic ring width, src/grid.cpp:85

struct Shape {
    int shape, ci, cj, hi, hj, rad;
};

__device__ bool in_footprint(const Shape& s, int i, int j) {
    if (s.shape == HK_OBSTACLE_RECTANGLE) return abs(i - s.ci) <= s.hi && abs(j - s.cj) <= s.hj;
    if (s.shape == HK_OBSTACLE_DISK) {
        const double di = i - s.ci, dj = j - s.cj;
        return di * di + dj * dj <= double(s.rad) * s.rad;
    }
    return false;
}

// New kind of cell (i, j); *overlap when the footprint or ring reaches the ghost frame.
__device__ uint8_t classify_one(const Shape& s, int nx, int ny, int i, int j, bool* overlap) {
    const bool ghost = i < kGhost || i >= nx - kGhost || j < kGhost || j >= ny - kGhost;
    *overlap = false;
    if (s.shape == HK_OBSTACLE_NONE) return ghost ? HK_CELL_GHOST : HK_CELL_INTERIOR;
    if (in_footprint(s, i, j)) {
        *overlap = ghost;
        return HK_CELL_OBSTACLE;
    }
    bool near = false;
    for (int dj = -kRing; dj <= kRing && !near; ++dj)
        for (int di = -kRing; di <= kRing && !near; ++di) near = in_footprint(s, i + di, j + dj);
    if (near) {
        *overlap = ghost;
        return HK_CELL_FORCED_RING;
    }
    return ghost ? HK_CELL_GHOST : HK_CELL_INTERIOR;
}

struct Fixed {
    double u[4];    // obstacle_state (conserved)
    double mom[5];  // obstacle_moments (rho, ux, uy, 0, T)
    bool ok;        // maxwellian(obstacle_moments) would not throw
};

struct Header {
    unsigned long long bad_config;  // first cell whose footprint/ring touches the ghost frame
    unsigned long long bad_cell;    // (cell << 8) | status of the reference's first throw in the loop
    int covered, vacated, nlist, pad;
};

// Pass 1: new classification (scratch) and the reference's failure point.
// apply = false: plain classify_cells straight into kind_out.
__global__ void obstacle_scan_kernel(Shape s, int nx, int ny, bool apply, uint8_t* __restrict__ kind_out,
                                     const uint8_t* __restrict__ kind_before, const int8_t* __restrict__ r,
                                     const double* __restrict__ hydro, double hr, Fixed fx, Header* __restrict__ h) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= (int64_t)nx * ny) return;
    const int i = int(c % nx), j = int(c / nx);
    bool overlap;
    const uint8_t after = classify_one(s, nx, ny, i, j, &overlap);
    kind_out[c] = after;
    if (overlap) atomicMin(&h->bad_config, (unsigned long long)c);
    if (!apply || after == HK_CELL_OBSTACLE) return;
    if (kind_before[c] == HK_CELL_OBSTACLE) {  // vacated: maxwellian(fixed_m)
        if (!fx.ok) atomicMin(&h->bad_cell, ((unsigned long long)c << 8) | HK_DEGENERATE);
        return;
    }
    if (after == HK_CELL_FORCED_RING && r[c] == 0) {  // pressure() then maxwellian()
        const double* u = hydro + 4 * c;
        int code = 0;
        if (!(u[0] > 0.0)) code = HK_POSITIVITY;
        else {
            const double p = (hr - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
            if (!(p > 0.0)) code = HK_POSITIVITY;
            else if (!(p / u[0] > 0.0)) code = HK_DEGENERATE;
        }
        if (code) atomicMin(&h->bad_cell, ((unsigned long long)c << 8) | (unsigned)code);
    }
}

// Pass 2: the loop body of apply_obstacle for every cell before the failure point.
__global__ void obstacle_apply_kernel(int64_t cells, const uint8_t* __restrict__ kind_new, uint8_t* __restrict__ kind,
                                      int8_t* __restrict__ r, double* __restrict__ hydro, double hr, Fixed fx,
                                      Header* __restrict__ h, int64_t* __restrict__ list_idx,
                                      double* __restrict__ list_mom) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cells || h->bad_config != ~0ull) return;
    const unsigned long long bad = h->bad_cell;
    const int64_t lim = bad == ~0ull ? cells : int64_t(bad >> 8);
    if (c > lim) return;
    const uint8_t before = kind[c], after = kind_new[c];
    double* u = hydro + 4 * c;
    if (c == lim) {  // the throwing cell: a vacated one has had r and hydro set first
        if (after != HK_CELL_OBSTACLE && before == HK_CELL_OBSTACLE) {
            r[c] = 2;
            for (int k = 0; k < 4; ++k) u[k] = fx.u[k];
        }
        return;
    }
    const double* m = nullptr;
    double mh[5];
    if (after == HK_CELL_OBSTACLE) {
        if (before != HK_CELL_OBSTACLE) atomicAdd(&h->covered, 1);
        for (int k = 0; k < 4; ++k) u[k] = fx.u[k];
        r[c] = 2;
    } else if (before == HK_CELL_OBSTACLE) {
        atomicAdd(&h->vacated, 1);
        r[c] = 2;
        for (int k = 0; k < 4; ++k) u[k] = fx.u[k];
        m = fx.mom;
    }
    if (after == HK_CELL_FORCED_RING && r[c] != 2) {
        if (r[c] == 0) {  // moments_from_conserved (src/coupling.cpp:7-13)
            const double p = (hr - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
            mh[0] = u[0];
            mh[1] = u[1] / u[0];
            mh[2] = u[2] / u[0];
            mh[3] = 0.0;
            mh[4] = p / u[0];
            m = mh;
        }
        r[c] = 2;
    }
    kind[c] = after;
    if (m) {
        const int k = atomicAdd(&h->nlist, 1);
        list_idx[k] = c;
        for (int q = 0; q < 5; ++q) list_mom[5 * k + q] = m[q];
    }
}

unsigned blocks_of(int64_t n) { return unsigned((n + 255) / 256); }

int check_spec(hk_ctx ctx, const hk_obstacle_spec* spec, int64_t nx, int64_t ny, const char* what) {
    if (!spec || nx < 1 || ny < 1 || nx * ny > (int64_t(1) << 40))
        return fail(ctx, HK_CONTRACT, std::string(what) + ": bad grid or null spec");
    if (spec->shape < HK_OBSTACLE_NONE || spec->shape > HK_OBSTACLE_DISK)
        return fail(ctx, HK_CONTRACT, std::string(what) + ": unknown obstacle shape");
    return HK_OK;
}

Shape shape_of(const hk_obstacle_spec* s) {
    return Shape{s->shape, s->center_i, s->center_j, s->half_i, s->half_j, s->radius};
}

}  // namespace
}  // namespace hk

using namespace hk;

extern "C" {

int hk_classify_cells(hk_ctx ctx, int64_t nx, int64_t ny, const hk_obstacle_spec* spec, uint8_t* kind_dev) {
    int st = check_spec(ctx, spec, nx, ny, "classify_cells");
    if (st) return st;
    cudaSetDevice(ctx->device);
    Header* h = nullptr;
    if (cudaMallocAsync(&h, sizeof(Header), ctx->stream) != cudaSuccess) return fail(ctx, HK_CUDA, "classify alloc");
    cudaMemsetAsync(h, 0xff, sizeof(Header), ctx->stream);
    const int64_t cells = nx * ny;
    obstacle_scan_kernel<<<blocks_of(cells), 256, 0, ctx->stream>>>(shape_of(spec), int(nx), int(ny), false, kind_dev,
                                                                     nullptr, nullptr, nullptr, 0.0, Fixed{}, h);
    ctx->launches++;
    Header hh;
    st = check_cuda(ctx, cudaGetLastError(), "classify kernel");
    if (!st) st = check_cuda(ctx, cudaMemcpyAsync(&hh, h, sizeof hh, cudaMemcpyDeviceToHost, ctx->stream), "classify");
    if (!st) st = check_cuda(ctx, cudaStreamSynchronize(ctx->stream), "classify");
    cudaFreeAsync(h, ctx->stream);
    if (!st && hh.bad_config != ~0ull)
        st = fail(ctx, HK_CONFIG, "obstacle or its forced-kinetic ring overlaps the ghost frame", (int64_t)hh.bad_config);
    return st;
}

int hk_apply_obstacle(hk_ctx ctx, int n, double vmax, hk_obstacle_spec* spec, int64_t nx, int64_t ny, int8_t* r_dev,
                      uint8_t* kind_dev, double* hydro_dev, double* f_dev, double heat_ratio, int* covered,
                      int* vacated) {
    HK_RANGE("hk_apply_obstacle");
    if (covered) *covered = 0;
    if (vacated) *vacated = 0;
    int st = check_spec(ctx, spec, nx, ny, "apply_obstacle");
    if (st) return st;
    if (spec->shape == HK_OBSTACLE_NONE) return HK_OK;
    if (n < 2 || n > 128) return fail(ctx, HK_UNSUPPORTED, "apply_obstacle: 2 <= n <= 128");
    cudaSetDevice(ctx->device);
    const bool moving = spec->move_di != 0 || spec->move_dj != 0;
    spec->center_i += spec->move_di;
    spec->center_j += spec->move_dj;

    // obstacle_moments / obstacle_state (src/coupling.cpp:39-53), host arithmetic
    Fixed fx{};
    const double T = spec->pressure / spec->rho;
    fx.mom[0] = spec->rho;
    fx.mom[1] = spec->ux;
    fx.mom[2] = spec->uy;
    fx.mom[3] = 0.0;
    fx.mom[4] = T;
    fx.u[0] = spec->rho;
    fx.u[1] = spec->rho * spec->ux;
    fx.u[2] = spec->rho * spec->uy;
    const double u2 = spec->ux * spec->ux + spec->uy * spec->uy + 0.0 * 0.0;
    fx.u[3] = spec->rho * T / (heat_ratio - 1.0) + 0.5 * spec->rho * u2;
    fx.ok = (spec->rho > 0.0) && (T > 0.0);

    const int64_t cells = nx * ny;
    const size_t off_kind = 64, off_idx = (off_kind + cells + 255) & ~size_t(255),
                 off_mom = off_idx + sizeof(int64_t) * cells, bytes = off_mom + sizeof(double) * 5 * cells;
    char* w = nullptr;
    if (cudaMallocAsync(&w, bytes, ctx->stream) != cudaSuccess) return fail(ctx, HK_CUDA, "apply_obstacle alloc");
    Header* h = reinterpret_cast<Header*>(w);
    uint8_t* kind_new = reinterpret_cast<uint8_t*>(w + off_kind);
    int64_t* list_idx = reinterpret_cast<int64_t*>(w + off_idx);
    double* list_mom = reinterpret_cast<double*>(w + off_mom);
    cudaMemsetAsync(h, 0xff, 2 * sizeof(unsigned long long), ctx->stream);
    cudaMemsetAsync(&h->covered, 0, 4 * sizeof(int), ctx->stream);
    obstacle_scan_kernel<<<blocks_of(cells), 256, 0, ctx->stream>>>(shape_of(spec), int(nx), int(ny), true, kind_new,
                                                                     kind_dev, r_dev, hydro_dev, heat_ratio, fx, h);
    obstacle_apply_kernel<<<blocks_of(cells), 256, 0, ctx->stream>>>(cells, kind_new, kind_dev, r_dev, hydro_dev,
                                                                      heat_ratio, fx, h, list_idx, list_mom);
    ctx->launches += 2;
    st = check_cuda(ctx, cudaGetLastError(), "obstacle kernels");
    // the list is empty when pass 1 found a ghost-frame overlap
    if (!st) st = maxwellian_launch(ctx, n, vmax, list_mom, cells, f_dev, nullptr, list_idx, &h->nlist);
    Header hh;
    if (!st) st = check_cuda(ctx, cudaMemcpyAsync(&hh, h, sizeof hh, cudaMemcpyDeviceToHost, ctx->stream), "obstacle");
    if (!st) st = check_cuda(ctx, cudaStreamSynchronize(ctx->stream), "obstacle");
    cudaFreeAsync(w, ctx->stream);
    if (st) return st;
    if (hh.bad_config != ~0ull)
        return moving ? fail(ctx, HK_SCENARIO_END, "moving obstacle left the domain", (int64_t)hh.bad_config)
                      : fail(ctx, HK_CONFIG, "obstacle or its forced-kinetic ring overlaps the ghost frame",
                             (int64_t)hh.bad_config);
    if (hh.bad_cell != ~0ull) {
        const int code = int(hh.bad_cell & 0xff);
        return fail(ctx, code,
                    code == HK_POSITIVITY ? "forced-ring cell: non-positive density or pressure"
                                          : "maxwellian requires positive density and temperature",
                    (int64_t)(hh.bad_cell >> 8));
    }
    if (covered) *covered = hh.covered;
    if (vacated) *vacated = hh.vacated;
    return HK_OK;
}

}  // extern "C"
