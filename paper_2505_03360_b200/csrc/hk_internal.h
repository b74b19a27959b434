// hk_internal.h — host-side objects behind the C-ABI handles.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hykin_b200.h"

// NVTX range over a C-ABI entry point (header-only NVTX 3; no cost unless a
// profiler attaches): nsys / ncu --nvtx show the library's calls by name.
#include <nvtx3/nvToolsExt.h>
struct HkRange {
    explicit HkRange(const char* name) { nvtxRangePushA(name); }
    ~HkRange() { nvtxRangePop(); }
    HkRange(const HkRange&) = delete;
    HkRange& operator=(const HkRange&) = delete;
};
#define HK_RANGE(name) HkRange hk_range_scope_(name)

struct hk_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    int64_t err_cell = -1;
    std::string err;
    int sm_count = 0;
    // scratch (grown on demand, never shrunk)
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    // pinned staging for the host entry points
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    std::map<int, int> max_clusters;  // key: kernel variant id
    // copy streams of the host (e2e) entry point: H2D / D2H overlap compute
    cudaStream_t s_in = nullptr, s_out = nullptr;
    // side stream of the N = 64 collision (guard + Nyquist correction beside the team kernel)
    cudaStream_t s_side = nullptr;
    // halo stream and halo buffers of the native x-slab IMEX steps (hk_steps.cu)
    cudaStream_t s_comm = nullptr;
    void* halo_work = nullptr;
    size_t halo_bytes = 0;
    // streamed-I/O flags for the next collision launch (host entry point), and
    // the guard's reroute list / count of the last launch (device pointers)
    const unsigned* sio_in_ready = nullptr;
    unsigned* sio_out_done = nullptr;
    int64_t sio_chunk = 0;
    bool sio_used = false;  // set by the launcher when the kernel honoured the flags
    unsigned* sio_flags = nullptr;  // cudaMalloc'd (stream memory ops reject pool memory)
    int64_t sio_flags_n = 0;
    int64_t* last_list = nullptr;
    int* last_count = nullptr;
    // lowest failing cell of the Euler / transition kernels (hk_euler.cu)
    void* bad_flag = nullptr;
    // work fields of the device-resident IMEX steps (hk_steps.cu)
    void* step_work = nullptr;
    size_t step_bytes = 0;
    // hybrid step workspaces (hk_hybrid.cu): per-cell arrays, kinetic batch + dense transport output
    void* hyb_small = nullptr;
    size_t hyb_small_bytes = 0;
    void* hyb_big = nullptr;
    size_t hyb_big_bytes = 0;
    // Nyquist-correction plane scratch (hk_nyqfix.cu)
    void* fix_scratch = nullptr;
    // N = 16 split-cell counters (hk_collision.cu), zeroed once and kept clean by the kernel
    unsigned* c16_ctr = nullptr;
    // padded x-slab of the native hybrid slab step (hk_hybrid.cu), grow-only
    void* slab_pad = nullptr;
    size_t slab_pad_bytes = 0;
    size_t fix_bytes = 0;
    // NCCL communicator (hk_comm.cu; ncclComm_t, loaded at run time)
    void* comm = nullptr;
    int nranks = 1, rank = 0;
    // optional CUDA-event timing of the collision kernels (tag -> event pairs)
    bool timing = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> events;
};

// Device-resident SpectralKernel (inc/spectral.hpp:15-33), re-laid out for
// coalesced loads by the collision kernels: tables are [entry][i1][i3][i2]
// with entry = distinct direction (the p = 0 row of src/spectral.cpp:83-90
// repeats e = (0,0,1) a2 times and is stored once with multiplicity a2).
struct hk_kernel_s {
    hk_ctx ctx = nullptr;
    int n = 0, a1 = 0, a2 = 0, md = 0;
    double vmax = 0, r_phys = 0, r = 0, jac = 0, weight = 0, mult0 = 1;
    double* alpha = nullptr;    // [md][n^3] exact radial weights
    double* alpha_p = nullptr;  // [md][n^3] exact planar weights
    double* loss = nullptr;     // [n^3] loss_diag (reference summation order)
    double2* wfast = nullptr;   // [md+1][n^3] Hermitian-symmetrised (alpha_s, alpha'_s); entry md = (loss_s, 0)
    double* abs_a = nullptr;    // [md][3][n][n] antisymmetric alpha on the Nyquist planes (signed)
    double* abs_ap = nullptr;   // [md][3][n][n] antisymmetric alpha' (signed)
    double absmax = 0;          // max over the abs tables (diagnostic)
};

namespace hk {

// Sets ctx->err and returns the status.
int fail(hk_ctx ctx, int status, const std::string& msg, int64_t cell = -1);
int check_cuda(hk_ctx ctx, cudaError_t e, const char* what);
// Ensures ctx->scratch holds >= bytes.
int ensure_scratch(hk_ctx ctx, size_t bytes);

// hk_weights.cu
int build_kernel_tables(hk_ctx ctx, hk_kernel k, const double* raw_alpha_dev,
                        const double* raw_alpha_p_dev, const double* raw_loss_dev);
int closed_form_raw_tables(hk_ctx ctx, hk_kernel k, double* raw_alpha_dev,
                           double* raw_alpha_p_dev, double* raw_loss_dev);

// hk_collision.cu
void preload_guard_kernels(int n);  // hk_collision.cu: load the kernels queued behind a streamed launch
int collision_launch(hk_ctx ctx, hk_kernel k, const double* f, double* q, int64_t ncells,
                     uint32_t flags, hk_cell_status* st);

// Event-timing helpers (no-ops unless ctx->timing).
void timing_begin(hk_ctx ctx, int tag);
void timing_end(hk_ctx ctx);

// hk_peak.cu
double fp64_peak(hk_ctx ctx);

// hk_comm.cu
void comm_destroy(hk_ctx ctx);
// Ghost columns of an x-slab field [ny][nx][cb bytes] into the padded copy
// [ny][nx + 2 w][cb] (columns [0, w) <- the left rank's last w, [w + nx, nx + 2 w)
// <- the right rank's first w; periodic over ranks), on the context stream: NCCL
// send/recv with a communicator of > 1 rank, else the slab's own wrap.
int halo_columns_padded(hk_ctx ctx, const void* src, size_t cb, int64_t nx, int64_t ny, int w, void* pad);

}  // namespace hk
