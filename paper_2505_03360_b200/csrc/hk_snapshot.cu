// hk_snapshot.cu — write_snapshot (the reference lists
// src/snapshot.cpp in its CMake but does not ship it).  Per call, in `dir`:
//   moments_<step>.csv  i,j,x,y,rho,ux,uy,T,P: one row per cell c = j nx + i,
//                       x = (i + 1/2) dx, y = (j + 1/2) dy;
//   regimes_<step>.txt  ny lines of nx layer numbers (0, 1, 2; -1 = obstacle);
//   meta_<step>.json    step, time, grid, velocity grid, the caller's config echo.
// Primitive moments: layer-0 cells from the conserved state (prim_from_conserved,
// src/coupling.cpp:24-31, pressure of src/euler.cpp:67-74), kinetic cells from
// moments_of(f) (prim_from_moments, src/coupling.cpp:33-35) on the device; P = rho T.
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hk_cells.cuh"
#include "hk_internal.h"

namespace hk {
namespace {

__global__ void prim_kernel(int64_t cells, const int8_t* __restrict__ r, const double* __restrict__ hydro,
                            const double* __restrict__ mom, const int* __restrict__ mst, double heat_ratio,
                            double* __restrict__ prim, int* __restrict__ bad) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cells) return;
    double* o = prim + c * 4;
    if (r[c] != 0) {
        const double* m = mom + c * 5;
        o[0] = m[0]; o[1] = m[1]; o[2] = m[2]; o[3] = m[4];
        if (mst[c] != HK_OK) atomicMin(bad, int(c));
    } else {
        const double* u = hydro + c * 4;
        const double p = (heat_ratio - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
        o[0] = u[0]; o[1] = u[1] / u[0]; o[2] = u[2] / u[0]; o[3] = p / u[0];
        if (!(u[0] > 0.0) || !(p > 0.0)) atomicMin(bad, int(c));
    }
}

}  // namespace
}  // namespace hk

using namespace hk;

extern "C" int hk_write_snapshot(hk_ctx ctx, int n, double vmax, int64_t nx, int64_t ny, double dx, double dy,
                                 const int8_t* r_dev, const uint8_t* kind_dev, const double* hydro_dev,
                                 const double* f_dev, double heat_ratio, int64_t step, double time, const char* dir,
                                 const char* config_json) {
    HK_RANGE("hk_write_snapshot");
    if (!ctx || !r_dev || !hydro_dev || !f_dev || !dir) return HK_CONTRACT;
    if (nx < 1 || ny < 1) return fail(ctx, HK_CONTRACT, "write_snapshot: empty grid");
    cudaSetDevice(ctx->device);
    const int64_t cells = nx * ny;
    int st;
    double *mom = nullptr, *prim = nullptr;
    int *mst = nullptr, *bad = nullptr;
    if ((st = check_cuda(ctx, cudaMallocAsync(&mom, sizeof(double) * 5 * cells, ctx->stream), "alloc")) ||
        (st = check_cuda(ctx, cudaMallocAsync(&prim, sizeof(double) * 4 * cells, ctx->stream), "alloc")) ||
        (st = check_cuda(ctx, cudaMallocAsync(&mst, sizeof(int) * (cells + 1), ctx->stream), "alloc")))
        return st;
    bad = mst + cells;
    const int big = 0x7fffffff;
    cudaMemcpyAsync(bad, &big, sizeof(int), cudaMemcpyHostToDevice, ctx->stream);
    // moments of every block (layer-0 blocks are ignored below)
    st = moments_launch(ctx, n, vmax, f_dev, cells, mom, nullptr, nullptr, nullptr, mst);
    if (!st) {
        prim_kernel<<<unsigned((cells + 255) / 256), 256, 0, ctx->stream>>>(cells, r_dev, hydro_dev, mom, mst, heat_ratio,
                                                                           prim, bad);
        ctx->launches++;
        st = check_cuda(ctx, cudaGetLastError(), "snapshot primitives");
    }
    std::vector<double> hp(size_t(cells) * 4);
    std::vector<int8_t> hr(cells);
    std::vector<uint8_t> hk(kind_dev ? cells : 0);
    int hbad = big;
    if (!st) st = check_cuda(ctx, cudaMemcpyAsync(hp.data(), prim, sizeof(double) * 4 * cells, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    if (!st) st = check_cuda(ctx, cudaMemcpyAsync(hr.data(), r_dev, cells, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    if (!st && kind_dev) st = check_cuda(ctx, cudaMemcpyAsync(hk.data(), kind_dev, cells, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    if (!st) st = check_cuda(ctx, cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
    if (!st) st = check_cuda(ctx, cudaStreamSynchronize(ctx->stream), "sync");
    cudaFreeAsync(mom, ctx->stream);
    cudaFreeAsync(prim, ctx->stream);
    cudaFreeAsync(mst, ctx->stream);
    if (st) return st;
    if (hbad != big)  // pressure / moments_of would throw (src/euler.cpp:68-72, src/moments.cpp:46-51)
        return fail(ctx, hr[hbad] != 0 ? HK_DEGENERATE : HK_POSITIVITY, "write_snapshot: non-physical state", hbad);
    const std::string base = std::string(dir) + "/";
    const std::string tag = std::to_string((long long)step);
    auto open = [&](const std::string& name) -> FILE* { return std::fopen((base + name).c_str(), "w"); };
    FILE* fm = open("moments_" + tag + ".csv");
    FILE* fr = open("regimes_" + tag + ".txt");
    FILE* fj = open("meta_" + tag + ".json");
    bool ok = fm && fr && fj;
    if (ok) {
        std::fprintf(fm, "i,j,x,y,rho,ux,uy,T,P\n");
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
                const double* p = hp.data() + 4 * (j * nx + i);
                std::fprintf(fm, "%lld,%lld,%.17g,%.17g,%.17g,%.17g,%.17g,%.17g,%.17g\n", (long long)i, (long long)j,
                             (i + 0.5) * dx, (j + 0.5) * dy, p[0], p[1], p[2], p[3], p[0] * p[3]);
            }
        for (int64_t j = 0; j < ny; ++j) {
            for (int64_t i = 0; i < nx; ++i) {
                const int64_t c = j * nx + i;
                const int v = (kind_dev && hk[c] == HK_CELL_OBSTACLE) ? -1 : int(hr[c]);
                std::fprintf(fr, i ? " %d" : "%d", v);
            }
            std::fputc('\n', fr);
        }
        std::fprintf(fj,
                     "{\"step\": %lld, \"time\": %.17g, \"nx\": %lld, \"ny\": %lld, \"dx\": %.17g, \"dy\": %.17g, "
                     "\"nv\": %d, \"vmax\": %.17g, \"heat_ratio\": %.17g, \"config\": %s}\n",
                     (long long)step, time, (long long)nx, (long long)ny, dx, dy, n, vmax, heat_ratio,
                     (config_json && *config_json) ? config_json : "null");
        ok = !std::ferror(fm) && !std::ferror(fr) && !std::ferror(fj);
    }
    const int e = errno;
    if (fm) ok = (std::fclose(fm) == 0) && ok;
    if (fr) ok = (std::fclose(fr) == 0) && ok;
    if (fj) ok = (std::fclose(fj) == 0) && ok;
    if (!ok) return fail(ctx, HK_IO, std::string("write_snapshot: cannot write into ") + dir + " (" + std::strerror(e) + ")");
    return HK_OK;
}
