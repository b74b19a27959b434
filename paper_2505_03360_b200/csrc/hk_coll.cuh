// hk_coll.cuh — arguments shared by the collision kernels (hk_collision.cu,
// hk_coll64.cu) and the N = 64 launcher.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "hk_internal.h"

namespace hk {

struct CollArgs {
    const double* f;
    double* q;
    int64_t ncells;
    const int64_t* list;    // optional cell list (rerouted cells)
    const int* list_count;  // device count for `list`
    const double* alpha;
    const double* alpha_p;
    const double* loss;
    const double2* wfast;
    int md;
    double mult0, jac, w;
    hk_cell_status* st;
    double2* nyq;      // [cell][3][N][N] F on the Nyquist planes (FAST: guard + correction) or null
    double2* xchg;     // [cluster][2 buffers][2 fields][C dest][P][N][N] L2 transpose scratch
    unsigned* team_ctr;  // [teams] barrier counters (team kernel), zeroed per launch
    unsigned long long* prof;  // optional [4]: producer spin, consumer spin, producer total, consumer total (cycles)
    // streamed host I/O (warp kernel): chunk c of `chunk` cells may be read once
    // in_ready[c] >= 1 (set by the H2D stream); out_done[c] counts finished
    // consumer-warp epilogues (the D2H stream waits for chunk * C * P).
    const unsigned* in_ready;
    unsigned* out_done;
    int64_t chunk;
};

// hk_coll64.cu: N = 64 team kernel (C = 32 CTAs per cell, cooperative launch).
// Bytes of exchange scratch per launch, and the launcher (exact = two complex
// transforms per direction, reference arithmetic; else the Hermitian-packed
// fast path that writes |F| on the Nyquist planes to args.nyq for the guard).
size_t coll64_xchg_bytes(hk_ctx ctx);
int launch_coll64(hk_ctx ctx, const CollArgs& args, bool exact, int64_t max_cells, int tag);

// hk_collgen.cu: the reference arithmetic for any n outside {16, 32, 64}
// (direct DFTs, chunked work fields); writes Q and the per-cell verdict.
int launch_coll_generic(hk_ctx ctx, hk_kernel k, const double* f, double* q, int64_t ncells, hk_cell_status* st);
__global__ void residue_kernel(int64_t ncells, hk_cell_status* st);

// hk_nyqfix.cu: exact Nyquist correction of the fast result for the cells on a
// device list (the guard's reroute list).
void nyq_fix_preload(int n);
void preload_guard_kernels(int n);
int nyq_fix_reserve(hk_ctx ctx, int n, int md, int64_t max_cells);
int launch_nyq_fix(hk_ctx ctx, int n, const int64_t* list, const int* count, int64_t max_cells, const double2* nyqF,
                   const double* ta, const double* tap, int md, double mult0, double jac, double w, double* q,
                   hk_cell_status* st);

}  // namespace hk
