// hk_cells.cuh — launchers of the per-cell and field kernels (hk_cells.cu, hk_field.cu).
#pragma once
#include "hk_internal.h"

namespace hk {

int moments_launch(hk_ctx ctx, int n, double vmax, const double* f, int64_t ncells, double* mom, double* sigma,
                   double* real, double* l1, int* status, const int64_t* src_idx = nullptr,
                   const int* count_dev = nullptr);
int maxwellian_launch(hk_ctx ctx, int n, double vmax, const double* mom, int64_t ncells, double* out, int* status,
                      const int64_t* dst_idx = nullptr, const int* count_dev = nullptr);
int stage_launch(hk_ctx ctx, bool esbgk, int n, double vmax, const double* fin, double* out, int64_t ncells, double a,
                 const double* eps_cell, double eps_scalar, double beta, double coeff, int* info, double* mom_out,
                 double* k1_out = nullptr, double k1_scale = 0.0);
// Stage solve of f* = f + cq q1 + ck k1 formed on the fly (the PR(2,2,2) second
// stage without a separate f_acc pass); stage_acc_supported(n): n a power of two >= 8.
bool stage_acc_supported(int n);
int stage_acc_launch(hk_ctx ctx, bool esbgk, int n, double vmax, const double* f, const double* q1, const double* k1,
                     double cq, double ck, double* out, int64_t ncells, double a, const double* eps_cell, double beta,
                     double coeff, int* info);
int residual_finish_launch(hk_ctx ctx, int n, double vmax, const double* f, double* q, int64_t ncells, double pen_coeff,
                           int* status);

// inc/moments.hpp:55-70 one operator at a time (hk_cells.cu)
int gaussian_launch(hk_ctx ctx, int n, double vmax, const double* mom, const double* theta, double beta,
                    int64_t ncells, double* out, int* fallback);
int match_launch(hk_ctx ctx, int n, double vmax, double* f, const double* target, int64_t ncells, int* status);
int remove_invariants_launch(hk_ctx ctx, int n, double vmax, double* q, const double* w, const double* uc,
                             int64_t ncells, int* status);

struct ClassifyParams {
    int nx, ny;
    double dx, dy, mu0, kappa0, eta0, eta1, delta0;
    int signed_sum;
};
int classify_launch(hk_ctx ctx, const ClassifyParams& p, const double* mom, const double* eps_cell, const double* l1,
                    const int8_t* r_in, int8_t* r_out, double* ind, int* status);

struct TransportParams {
    int n;
    double vmax;
    int nx, ny;      // output (interior) cells
    int x_halo;      // 0: periodic in x; >= 2: input carries x_halo ghost columns per side;
                     // -2: ghost columns come from the lh / rh slabs below
    double dx, dy, eps_weno;
    // x_halo == -2: lh / rh are [ny][lnx][n^3] / [ny][rnx][n^3] slabs whose LAST two /
    // FIRST two columns are the ghosts: 2 for separate halo buffers, the neighbour's
    // nx when lh / rh point straight at the neighbour rank's slab (NVLink peer memory)
    int lnx = 2, rnx = 2;
    // optional row activity of the output strips (lane-per-column kernel only),
    // [strips][ny] from transport_row_activity: rows of a strip with no cell of
    // interest are skipped (their outputs are left unwritten)
    const uint8_t* row_act = nullptr;
    // optional compact output (lane-per-column kernel, plain T only): cell c's
    // result goes to out + out_pos[c] n^3, cells with out_pos[c] < 0 are not written
    const int* out_pos = nullptr;
    // optional batch-resident input (lane kernel, x_halo == 0): cells with in_pos[c] >= 0
    // are read from in_batch + in_pos[c] n^3, the others from the dense field
    const int* in_pos = nullptr;
    const double* in_batch = nullptr;
};

// Final PR(2,2,2) combination fused into the second transport of a step
// (src/boltzmann.cpp:99-108, src/esbgk.cpp:90-97): with T = T(Y2) computed in
// place,  q2 = T + res/eps,  f_acc = f + dt a_ex10 q1 + a_im10 k1,
// k2 = (Y2 - f_acc)/a_im11,  f += dt (w0 q1 + w1 q2) + w0 k1 + w1 k2.
// Elementwise PR(2,2,2) work fused into a transport sweep T(y) (hk_transport.cu).
//   mode 1: f <- f + dt (w_ex0 q1 + w_ex1 q2) + w_im0 k1 + w_im1 k2, q2 = T(y) + res / eps,
//           k2 = (y - f_acc) / a_im11, f_acc = f + dt a_ex10 q1 + a_im10 k1   (src/boltzmann.cpp:80-105)
//   mode 2: y = Y1, q1 = T(Y1) + res / eps, k1 = (Y1 - f) k1_scale:
//           fa <- f_acc,  f <- G = f + dt w_ex0 q1 + w_im0 k1 - (w_im1 / a_im11) f_acc
//   mode 3: y = Y2 (the stage of f_acc):  f <- G + dt w_ex1 q2 + (w_im1 / a_im11) Y2
// Modes 2 + 3 are mode 1 regrouped: the final update is linear in (f, q1, k1),
// so the transport of Y1 folds those three fields into two (f_acc for the
// second stage, G in place of f) and neither q1 nor k1 is ever stored.
struct FinalCombine {
    double* f;               // in/out
    const double* q1;
    const double* k1;
    const double* res;       // nullable (ES-BGK)
    const double* eps;       // per cell
    double dt, a_ex10, a_im10, a_im11, w_ex0, w_ex1, w_im0, w_im1;
    int mode = 1;
    double* fa = nullptr;    // mode 2: f_acc out
    double k1_scale = 0.0;   // mode 2: 1 / a_im00
};
// true when transport_launch takes the lane-per-column sweep for these shapes (out_pos honoured)
bool transport_lanes_path(const TransportParams& p);
int transport_launch(hk_ctx ctx, const TransportParams& p, const double* f, double* out, const double* lh = nullptr,
                     const double* rh = nullptr);
// hk_transport.cu: y-marching transport (n a power of two, n^3 % 32 == 0, ny >= 3)
int transport_march_launch(hk_ctx ctx, const TransportParams& p, int lg, const double* f, double* out, const double* lh,
                           const double* rh, const FinalCombine* fin = nullptr);
// PR(2,2,2) second transport + final combination (x periodic); false if the
// marching kernel does not apply (caller runs transport + combine instead).
bool transport_final_supported(const TransportParams& p);
int transport_fused_launch(hk_ctx ctx, const TransportParams& p, const double* y, const FinalCombine& fc,
                           const double* lh = nullptr, const double* rh = nullptr);
// Row activity of the transport strips for a [ny][nx] cell mask (nonzero = the
// output is needed); act holds transport_row_activity_bytes(nx, ny) bytes.
size_t transport_row_activity_bytes(int nx, int ny);
int transport_row_activity(hk_ctx ctx, int nx, int ny, const int8_t* mask, uint8_t* act);
int transport_final_launch(hk_ctx ctx, const TransportParams& p, const double* y2, const FinalCombine& fc);
int combine_launch(hk_ctx ctx, int op, int64_t count, int64_t nb, double dt, const double* eps, double* o,
                   const double* f, const double* y, const double* q1, const double* k1, const double* tr,
                   const double* res);

// out = x + a*y + b*z (elementwise, any of y/z nullable)
int axpby_launch(hk_ctx ctx, int64_t count, double* out, const double* x, double a, const double* y, double b,
                 const double* z);

}  // namespace hk
