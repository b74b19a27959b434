// hk_steps.cu — C-ABI entries for the per-cell / field operators and the
// device-resident PR(2,2,2) IMEX steps (include/hykin_b200.h).
//
//   penalized_imex_step   src/boltzmann.cpp:47-110
//   esbgk_imex_step       src/esbgk.cpp:47-99
//   ImexTableau::pr222    inc/imex.hpp:23-34
// All buffers stay in HBM; one step is a fixed sequence of stream-ordered
// launches (CUDA-graph capturable).
#include <cmath>

#include "hk_cells.cuh"
#include "hk_common.cuh"
#include "hk_internal.h"

namespace hk {

namespace {

struct PR222 {
    double a_ex10, a_im00, a_im10, a_im11, w_ex0, w_ex1, w_im0, w_im1;
};
PR222 pr222() {
    const double C = 1.0 / std::sqrt(2.0);
    const double delta = 1.0 - 1.0 / (2.0 * C);
    return {1.0, 1.0 - C, C - delta, delta, 0.5, 0.5, 0.5, 0.5};
}

// Fused elementwise IMEX combinations; e = per-cell Knudsen number.
enum CombOp { K1 = 0, Q1 = 1, FACC = 2, FINAL = 3 };

__global__ void combine_kernel(int op, int64_t count, int64_t nb, PR222 t, double dt, const double* __restrict__ e,
                               double* __restrict__ o, const double* __restrict__ f, const double* __restrict__ y,
                               const double* __restrict__ q1, const double* __restrict__ k1,
                               const double* __restrict__ tr, const double* __restrict__ res) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double inv_eps = res ? 1.0 / e[i / nb] : 0.0;
        switch (op) {
        case K1:  // k1 = (Y - f) / a11   (src/boltzmann.cpp:65-67)
            o[i] = (y[i] - f[i]) * (1.0 / t.a_im00);
            break;
        case Q1:  // q1 = T(Y) + res(Y) / eps   (:69-76)
            o[i] = res ? tr[i] + res[i] * inv_eps : tr[i];
            break;
        case FACC:  // f_acc = f + dt a_ex10 q1 + a_im10 k1   (:80-81)
            o[i] = f[i] + dt * t.a_ex10 * q1[i] + t.a_im10 * k1[i];
            break;
        default: {  // final streaming combination (:99-108)
            const double q2k = res ? tr[i] + res[i] * inv_eps : tr[i];
            const double fc = o[i];
            const double facc = fc + dt * t.a_ex10 * q1[i] + t.a_im10 * k1[i];
            const double k2 = (y[i] - facc) * (1.0 / t.a_im11);
            o[i] = fc + (dt * (t.w_ex0 * q1[i] + t.w_ex1 * q2k) + t.w_im0 * k1[i] + t.w_im1 * k2);
        }
        }
    }
}

int combine(hk_ctx ctx, int op, int64_t count, int64_t nb, const PR222& t, double dt, const double* e, double* o,
            const double* f, const double* y, const double* q1, const double* k1, const double* tr, const double* res) {
    const int64_t blocks = (count + 255) / 256, cap = int64_t(ctx->sm_count) * 16;
    combine_kernel<<<unsigned(blocks < cap ? blocks : cap), 256, 0, ctx->stream>>>(op, count, nb, t, dt, e, o, f, y, q1,
                                                                                   k1, tr, res);
    ctx->launches++;
    return check_cuda(ctx, cudaGetLastError(), "combine kernel");
}

struct Work {
    double *y, *q1, *k1, *tr, *res, *fa;
};

// Work fields of a step: the caller's buffer, else a context-owned one kept
// across steps (grow-only; re-allocating ~100 GB per step costs seconds).
int get_work(hk_ctx ctx, double* user, int64_t count, Work& w, double** owned, int nfields = 6) {
    *owned = nullptr;
    double* base = user;
    if (!base) {
        const size_t need = sizeof(double) * count * nfields;
        if (need > ctx->step_bytes) {
            if (ctx->step_work) {
                cudaStreamSynchronize(ctx->stream);
                cudaFree(ctx->step_work);
                ctx->step_work = nullptr;
                ctx->step_bytes = 0;
            }
            int st = check_cuda(ctx, cudaMalloc(&ctx->step_work, need), "step work alloc");
            if (st) return st;
            ctx->step_bytes = need;
        }
        base = static_cast<double*>(ctx->step_work);
    }
    if (nfields == 3)  // the regrouped step: Y, f_acc, residual
        w = {base, nullptr, nullptr, nullptr, base + 2 * count, base + count};
    else
        w = {base, base + count, base + 2 * count, base + 3 * count, base + 4 * count, base + 5 * count};
    return HK_OK;
}

}  // namespace

int combine_launch(hk_ctx ctx, int op, int64_t count, int64_t nb, double dt, const double* eps, double* o,
                   const double* f, const double* y, const double* q1, const double* k1, const double* tr,
                   const double* res) {
    if (op < 0 || op > 3) return fail(ctx, HK_CONTRACT, "combine: op in 0..3");
    return combine(ctx, op, count, nb, pr222(), dt, eps, o, f, y, q1, k1, tr, res);
}

}  // namespace hk

using namespace hk;

extern "C" {

int hk_moments_batch(hk_ctx ctx, int n, double vmax, const double* f_dev, int64_t ncells, double* mom_dev,
                     double* sigma_dev, double* real_dev, double* l1_dev, int* status_dev) {
    HK_RANGE("hk_moments_batch");
    cudaSetDevice(ctx->device);
    return moments_launch(ctx, n, vmax, f_dev, ncells, mom_dev, sigma_dev, real_dev, l1_dev, status_dev);
}

int hk_maxwellian_batch(hk_ctx ctx, int n, double vmax, const double* mom_dev, int64_t ncells, double* out_dev,
                        int* status_dev) {
    HK_RANGE("hk_maxwellian_batch");
    cudaSetDevice(ctx->device);
    return maxwellian_launch(ctx, n, vmax, mom_dev, ncells, out_dev, status_dev);
}

int hk_anisotropic_gaussian_batch(hk_ctx ctx, int n, double vmax, const double* mom_dev, const double* theta_dev,
                                  double beta, int64_t ncells, double* out_dev, int* fallback_dev) {
    HK_RANGE("hk_anisotropic_gaussian_batch");
    cudaSetDevice(ctx->device);
    return gaussian_launch(ctx, n, vmax, mom_dev, theta_dev, beta, ncells, out_dev, fallback_dev);
}

int hk_match_moments_batch(hk_ctx ctx, int n, double vmax, double* f_dev, const double* target_dev, int64_t ncells,
                           int* status_dev) {
    HK_RANGE("hk_match_moments_batch");
    cudaSetDevice(ctx->device);
    return match_launch(ctx, n, vmax, f_dev, target_dev, ncells, status_dev);
}

int hk_remove_invariant_moments_batch(hk_ctx ctx, int n, double vmax, double* q_dev, const double* weight_dev,
                                      const double* uc_dev, int64_t ncells, int* status_dev) {
    HK_RANGE("hk_remove_invariant_moments_batch");
    cudaSetDevice(ctx->device);
    return remove_invariants_launch(ctx, n, vmax, q_dev, weight_dev, uc_dev, ncells, status_dev);
}

int hk_esbgk_stage_batch(hk_ctx ctx, int n, double vmax, const double* f_star_dev, double* out_dev, int64_t ncells,
                         double a, const double* eps_dev, double eps, double beta, double nu_coeff, int* info_dev,
                         double* mom_dev) {
    HK_RANGE("hk_esbgk_stage_batch");
    cudaSetDevice(ctx->device);
    return stage_launch(ctx, true, n, vmax, f_star_dev, out_dev, ncells, a, eps_dev, eps, beta, nu_coeff, info_dev,
                        mom_dev);
}

int hk_penalized_stage_batch(hk_ctx ctx, int n, double vmax, const double* f_star_dev, double* out_dev,
                             int64_t ncells, double a, const double* eps_dev, double eps, double pen_coeff,
                             int* info_dev, double* mom_dev) {
    HK_RANGE("hk_penalized_stage_batch");
    cudaSetDevice(ctx->device);
    return stage_launch(ctx, false, n, vmax, f_star_dev, out_dev, ncells, a, eps_dev, eps, 0.0, pen_coeff, info_dev,
                        mom_dev);
}

int hk_penalized_residual_batch(hk_ctx ctx, hk_kernel k, const double* f_dev, double* out_dev, int64_t ncells,
                                double pen_coeff, uint32_t flags, int* status_dev, hk_cell_status* st_dev) {
    HK_RANGE("hk_penalized_residual_batch");
    cudaSetDevice(ctx->device);
    int st = hk_collision_batch(ctx, k, f_dev, out_dev, ncells, flags & ~HK_COLL_STRICT, st_dev);
    if (st) return st;
    return residual_finish_launch(ctx, k->n, k->vmax, f_dev, out_dev, ncells, pen_coeff, status_dev);
}

int hk_classify(hk_ctx ctx, int nx, int ny, double dx, double dy, const double* mom_dev, const double* eps_dev,
                const double* l1_dev, const int8_t* r_in_dev, int8_t* r_out_dev, double* ind_dev, int* status_dev,
                double eta0, double eta1, double delta0, double mu0, double kappa0, int signed_sum) {
    HK_RANGE("hk_classify");
    cudaSetDevice(ctx->device);
    if (!(eta0 > 0.0) || !(eta1 > 0.0) || !(delta0 > 0.0))  // Thresholds::validate (src/indicators.cpp:9-12)
        return fail(ctx, HK_CONFIG, "regime thresholds eta0, eta1, delta0 must be positive");
    ClassifyParams p{nx, ny, dx, dy, mu0, kappa0, eta0, eta1, delta0, signed_sum};
    return classify_launch(ctx, p, mom_dev, eps_dev, l1_dev, r_in_dev, r_out_dev, ind_dev, status_dev);
}

int hk_transport_rhs(hk_ctx ctx, int n, double vmax, const double* f_dev, double* out_dev, int nx, int ny,
                     int x_halo, double dx, double dy, double eps_weno) {
    HK_RANGE("hk_transport_rhs");
    cudaSetDevice(ctx->device);
    TransportParams p{n, vmax, nx, ny, x_halo, dx, dy, eps_weno};
    return transport_launch(ctx, p, f_dev, out_dev);
}

// Shared driver of both PR(2,2,2) steps on a periodic all-kinetic field.
static int imex_step(hk_ctx ctx, hk_kernel k, bool boltz, int n, double vmax, double* f, int nx, int ny, double dx,
                     double dy, double dt, const double* eps_dev, double beta, double coeff, double eps_weno,
                     uint32_t flags, double* work_dev, bool slab = false) {
    cudaSetDevice(ctx->device);
    const int64_t cells = (int64_t)nx * ny, nb = (int64_t)n * n * n, count = cells * nb;
    const PR222 t = pr222();
    TransportParams tps{n, vmax, nx, ny, slab ? -2 : 0, dx, dy, eps_weno};
    // the regrouped step (below) needs 3 work fields (Y, f_acc, residual), the general one 6
    const bool regroup = stage_acc_supported(n) && transport_final_supported(tps);
    Work w;
    double* owned = nullptr;
    int st = get_work(ctx, work_dev, count, w, &owned, regroup ? 3 : 6);
    if (st) return st;
    // x-slab: the two [ny][2][n^3] halo buffers (context-owned, grow-only)
    double *lh = nullptr, *rh = nullptr;
    if (slab) {
        const size_t need = sizeof(double) * 4 * (size_t)ny * nb;
        if (need > ctx->halo_bytes) {
            if (ctx->halo_work) {
                cudaStreamSynchronize(ctx->stream);
                cudaFree(ctx->halo_work);
                ctx->halo_work = nullptr;
                ctx->halo_bytes = 0;
            }
            if ((st = check_cuda(ctx, cudaMalloc(&ctx->halo_work, need), "halo buffers"))) return st;
            ctx->halo_bytes = need;
        }
        lh = static_cast<double*>(ctx->halo_work);
        rh = lh + 2 * (int64_t)ny * nb;
    }
    TransportParams tp{n, vmax, nx, ny, 0, dx, dy, eps_weno};
    auto stage = [&](const double* fin, double a, double* out, double* k1) {
        return boltz ? stage_launch(ctx, false, n, vmax, fin, out, cells, a, eps_dev, 0.0, 0.0, coeff, nullptr, nullptr,
                                    k1, 1.0 / t.a_im00)
                     : stage_launch(ctx, true, n, vmax, fin, out, cells, a, eps_dev, 0.0, beta, coeff, nullptr, nullptr,
                                    k1, 1.0 / t.a_im00);
    };
    auto residual = [&](const double* y, double* out) {
        int s = hk_collision_batch(ctx, k, y, out, cells, flags & ~HK_COLL_STRICT, nullptr);
        return s ? s : residual_finish_launch(ctx, n, vmax, y, out, cells, coeff, nullptr);
    };
    // x-slab halos of the stage field y: issued on the comm stream as soon as the
    // stage is written, overlapped with the residual (collision) on the main
    // stream; the transport waits for them.  With a communicator of >1 rank the
    // two edge columns travel over NCCL (hk_halo_exchange); otherwise the slab is
    // its own periodic neighbour (local copies).
    cudaEvent_t ev_y = nullptr, ev_h = nullptr;
    if (slab) {
        if (!ctx->s_comm &&
            (st = check_cuda(ctx, cudaStreamCreateWithFlags(&ctx->s_comm, cudaStreamNonBlocking), "comm stream")))
            return st;
        cudaEventCreateWithFlags(&ev_y, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ev_h, cudaEventDisableTiming);
    }
    auto halo_begin = [&](const double* y) -> int {
        if (!slab) return HK_OK;
        cudaEventRecord(ev_y, ctx->stream);
        cudaStreamWaitEvent(ctx->s_comm, ev_y, 0);
        int e;
        if (ctx->comm && ctx->nranks > 1) {
            cudaStream_t main_s = ctx->stream;
            ctx->stream = ctx->s_comm;
            e = hk_halo_exchange(ctx, n, y, nx, ny, lh, rh);
            ctx->stream = main_s;
        } else {
            const size_t rowb = sizeof(double) * nx * nb, twob = sizeof(double) * 2 * nb;
            e = check_cuda(ctx, cudaMemcpy2DAsync(lh, twob, y + (nx - 2) * nb, rowb, twob, ny, cudaMemcpyDeviceToDevice,
                                                  ctx->s_comm), "halo copy");
            if (!e)
                e = check_cuda(ctx, cudaMemcpy2DAsync(rh, twob, y, rowb, twob, ny, cudaMemcpyDeviceToDevice, ctx->s_comm),
                               "halo copy");
        }
        cudaEventRecord(ev_h, ctx->s_comm);
        return e;
    };
    auto transport = [&](const double* y, double* out) -> int {
        if (!slab) return transport_launch(ctx, tp, y, out);
        cudaStreamWaitEvent(ctx->stream, ev_h, 0);
        TransportParams ts = tp;
        ts.x_halo = -2;
        return transport_launch(ctx, ts, y, out, lh, rh);
    };
    double* R = boltz ? w.res : nullptr;
    auto timed = [&](int tag, auto&& fn) {  // hk_ctx_set_timing: per-part step times (tags 10..13)
        timing_begin(ctx, tag);
        const int e = fn();
        timing_end(ctx);
        return e;
    };
    if (regroup) {
        // Regrouped step (FinalCombine modes 2 / 3): four field kernels, and
        // neither q1 nor k1 is stored.  T(Y1) writes f_acc and, in place of f,
        // G = f + dt w_ex0 q1 + w_im0 k1 - (w_im1 / a_im11) f_acc; T(Y2) finishes
        // f = G + dt w_ex1 q2 + (w_im1 / a_im11) Y2, which is the reference's
        // final update (src/boltzmann.cpp:100-105, src/esbgk.cpp:92-97) with
        // k2 = (Y2 - f_acc) / a_im11 expanded.
        FinalCombine fm{f, nullptr, nullptr, R, eps_dev, dt, t.a_ex10, t.a_im10, t.a_im11, t.w_ex0, t.w_ex1, t.w_im0,
                        t.w_im1};
        fm.fa = w.fa;
        fm.k1_scale = 1.0 / t.a_im00;
        auto fused = [&](const double* y, int mode) -> int {
            fm.mode = mode;
            if (slab) cudaStreamWaitEvent(ctx->stream, ev_h, 0);
            return transport_fused_launch(ctx, tps, y, fm, lh, rh);
        };
        if (!st) st = timed(10, [&] { return stage(f, t.a_im00 * dt, w.y, nullptr); });  // Y1
        if (!st) st = halo_begin(w.y);
        if (!st && boltz) st = residual(w.y, w.res);                                     // res(Y1), overlaps the halos
        if (!st) st = timed(11, [&] { return fused(w.y, 2); });                          // T(Y1) -> f_acc, G
        if (!st) st = timed(12, [&] { return stage(w.fa, t.a_im11 * dt, w.y, nullptr); });  // Y2
        if (!st) st = halo_begin(w.y);
        if (!st && boltz) st = residual(w.y, w.res);                                     // res(Y2)
        if (!st) st = timed(13, [&] { return fused(w.y, 3); });                          // T(Y2) -> f
        if (slab) {
            cudaStreamWaitEvent(ctx->stream, ev_h, 0);
            cudaEventDestroy(ev_y);
            cudaEventDestroy(ev_h);
        }
        if (owned) cudaFreeAsync(owned, ctx->stream);
        return st;
    }
    // Stage 1 (k1 fused into the stage kernel), explicit q1; ES-BGK has no
    // residual, so T(Y1) is q1 itself.
    if (!st) st = timed(10, [&] { return stage(f, t.a_im00 * dt, w.y, w.k1); });            // Y1, k1
    if (!st) st = halo_begin(w.y);
    if (!st && boltz) st = residual(w.y, w.res);                                           // res(Y1), overlaps the halos
    if (!st) st = timed(11, [&] { return transport(w.y, boltz ? w.tr : w.q1); });           // T(Y1)
    if (!st && boltz) st = combine(ctx, Q1, count, nb, t, dt, eps_dev, w.q1, 0, 0, 0, 0, w.tr, R);  // q1
    if (stage_acc_supported(n)) {  // Y2 = stage(f_acc), f_acc = f + dt a_ex10 q1 + a_im10 k1 formed in the stage
        if (!st)
            st = timed(12, [&] {
                return stage_acc_launch(ctx, !boltz, n, vmax, f, w.q1, w.k1, dt * t.a_ex10, t.a_im10, w.y, cells,
                                        t.a_im11 * dt, eps_dev, boltz ? 0.0 : beta, coeff, nullptr);
            });
    } else {
        if (!st) st = combine(ctx, FACC, count, nb, t, dt, eps_dev, w.fa, f, 0, w.q1, w.k1, 0, 0);  // f_acc
        if (!st) st = stage(w.fa, t.a_im11 * dt, w.y, nullptr);                                // Y2
    }
    if (!st) st = halo_begin(w.y);
    if (!st && boltz) st = residual(w.y, w.res);                                           // res(Y2)
    if (!st && !slab && transport_final_supported(tp)) {  // T(Y2) + final combination, one kernel
        const FinalCombine fc{f, w.q1, w.k1, R, eps_dev, dt, t.a_ex10, t.a_im10, t.a_im11, t.w_ex0, t.w_ex1, t.w_im0,
                              t.w_im1};
        st = timed(13, [&] { return transport_final_launch(ctx, tp, w.y, fc); });
    } else {
        if (!st) st = timed(13, [&] { return transport(w.y, w.tr); });                      // T(Y2)
        if (!st) st = combine(ctx, FINAL, count, nb, t, dt, eps_dev, f, 0, w.y, w.q1, w.k1, w.tr, R);
    }
    if (slab) {
        cudaStreamWaitEvent(ctx->stream, ev_h, 0);  // error paths: the comm stream's copies are done before reuse
        cudaEventDestroy(ev_y);
        cudaEventDestroy(ev_h);
    }
    if (owned) cudaFreeAsync(owned, ctx->stream);
    return st;
}

int hk_esbgk_imex_step(hk_ctx ctx, int n, double vmax, double* f_dev, int nx, int ny, double dx, double dy, double dt,
                       const double* eps_dev, double beta, double nu_coeff, double eps_weno, double* work_dev) {
    HK_RANGE("hk_esbgk_imex_step");
    return imex_step(ctx, nullptr, false, n, vmax, f_dev, nx, ny, dx, dy, dt, eps_dev, beta, nu_coeff, eps_weno, 0,
                     work_dev);
}

int hk_penalized_imex_step(hk_ctx ctx, hk_kernel k, double* f_dev, int nx, int ny, double dx, double dy, double dt,
                           const double* eps_dev, double pen_coeff, double eps_weno, uint32_t flags,
                           double* work_dev) {
    HK_RANGE("hk_penalized_imex_step");
    return imex_step(ctx, k, true, k->n, k->vmax, f_dev, nx, ny, dx, dy, dt, eps_dev, 0.0, pen_coeff, eps_weno, flags,
                     work_dev);
}

int hk_transport_rhs_peer(hk_ctx ctx, int n, double vmax, const double* f_dev, const double* left_slab_dev,
                          int left_nx, const double* right_slab_dev, int right_nx, double* out_dev, int nx, int ny,
                          double dx, double dy, double eps_weno) {
    HK_RANGE("hk_transport_rhs_peer");
    if (left_nx < 2 || right_nx < 2 || !left_slab_dev || !right_slab_dev)
        return fail(ctx, HK_CONTRACT, "transport_rhs_peer: neighbour slabs need >= 2 columns");
    cudaSetDevice(ctx->device);
    TransportParams p{n, vmax, nx, ny, -2, dx, dy, eps_weno};
    p.lnx = left_nx;
    p.rnx = right_nx;
    return transport_launch(ctx, p, f_dev, out_dev, left_slab_dev, right_slab_dev);
}

int hk_transport_rhs_slab(hk_ctx ctx, int n, double vmax, const double* f_dev, const double* left_dev,
                          const double* right_dev, double* out_dev, int nx, int ny, double dx, double dy,
                          double eps_weno) {
    HK_RANGE("hk_transport_rhs_slab");
    cudaSetDevice(ctx->device);
    TransportParams p{n, vmax, nx, ny, -2, dx, dy, eps_weno};
    return transport_launch(ctx, p, f_dev, out_dev, left_dev, right_dev);
}

int hk_imex_combine(hk_ctx ctx, int op, int64_t count, int64_t nb, double dt, const double* eps_dev, double* out_dev,
                    const double* f_dev, const double* y_dev, const double* q1_dev, const double* k1_dev,
                    const double* tr_dev, const double* res_dev) {
    cudaSetDevice(ctx->device);
    return combine_launch(ctx, op, count, nb, dt, eps_dev, out_dev, f_dev, y_dev, q1_dev, k1_dev, tr_dev, res_dev);
}

int hk_axpby(hk_ctx ctx, int64_t count, double* out_dev, const double* x_dev, double a, const double* y_dev, double b,
             const double* z_dev) {
    cudaSetDevice(ctx->device);
    return axpby_launch(ctx, count, out_dev, x_dev, a, y_dev, b, z_dev);
}

}  // extern "C"

extern "C" {

int hk_penalized_imex_step_slab(hk_ctx ctx, hk_kernel k, double* f_dev, int nx_local, int ny, double dx, double dy,
                                double dt, const double* eps_dev, double pen_coeff, double eps_weno, uint32_t flags,
                                double* work_dev) {
    HK_RANGE("hk_penalized_imex_step_slab");
    if (!ctx || !k) return HK_CONTRACT;
    if (nx_local < 2 || ny < 1) return fail(ctx, HK_CONTRACT, "slab step: need nx_local >= 2 columns");
    return imex_step(ctx, k, true, k->n, k->vmax, f_dev, nx_local, ny, dx, dy, dt, eps_dev, 0.0, pen_coeff, eps_weno,
                     flags, work_dev, true);
}

int hk_esbgk_imex_step_slab(hk_ctx ctx, int n, double vmax, double* f_dev, int nx_local, int ny, double dx, double dy,
                            double dt, const double* eps_dev, double beta, double nu_coeff, double eps_weno,
                            double* work_dev) {
    HK_RANGE("hk_esbgk_imex_step_slab");
    if (!ctx) return HK_CONTRACT;
    if (nx_local < 2 || ny < 1) return fail(ctx, HK_CONTRACT, "slab step: need nx_local >= 2 columns");
    return imex_step(ctx, nullptr, false, n, vmax, f_dev, nx_local, ny, dx, dy, dt, eps_dev, beta, nu_coeff, eps_weno, 0,
                     work_dev, true);
}

}  // extern "C"
