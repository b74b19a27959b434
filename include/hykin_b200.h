/*
 * hykin_b200.h — C-ABI of the B200-native fast-spectral collision path.
 *
 * Drop-in boundary for the data-parallel hot path of the reference solver
 * (`hykin`, /root/reference/proj/core).  Each entry point names the
 * reference interface it replaces (file:line, include/hykin = inc/).  The
 * reference exposes C++ free functions taking std::span and throwing
 * hykin::error subclasses; this ABI takes plain pointers + sizes and
 * returns status codes that map 1:1 onto those exception classes
 * (inc/errors.hpp:9-61).  INTEGRATION.md shows the C++ / ctypes bindings a
 * maintainer adds on the reference side.
 *
 * Layout contract (replaces DistributionField, inc/fields.hpp:48-79): a
 * field is ONE contiguous cell-major slab of doubles,
 *     f[cell][k1][k2][k3],  cell = j*nx + i (inc/grid.hpp:30),
 *     k index (k1*n + k2)*n + k3 (inc/grid.hpp:54), 64-bit offsets.
 * `*_dev` pointers are CUDA device pointers; `*_host` pointers are host
 * memory (pageable or pinned).  All device calls are ordered on the
 * context's stream; only calls that return per-cell verdicts synchronise.
 * fp64 throughout.  No CPU fallback: without a usable sm_100 device every
 * call returns HK_CUDA.
 */
#ifndef HYKIN_B200_H
#define HYKIN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes == exception classes of inc/errors.hpp. */
typedef enum {
    HK_OK = 0,
    HK_CONFIG = 1,                /* hykin::config_error */
    HK_ALIASING = 2,              /* hykin::aliasing_config_error */
    HK_DEGENERATE = 3,            /* hykin::degenerate_state_error */
    HK_NUMERICAL_CONSISTENCY = 4, /* hykin::numerical_consistency_error */
    HK_CONTRACT = 5,              /* hykin::contract_violation */
    HK_CUDA = 6,                  /* device / runtime failure (no reference analogue) */
    HK_NCCL = 7,                  /* collective failure (no reference analogue) */
    HK_POSITIVITY = 8,            /* hykin::positivity_error */
    HK_UNSUPPORTED = 9,           /* size not implemented on this path */
    HK_SCENARIO_END = 10,         /* hykin::scenario_end_error */
    HK_IO = 11                    /* hykin::io_error */
} hk_status;

/* Per-cell verdict written by the collision kernels (device or host array). */
typedef struct {
    double max_re;    /* max_k |Re Q_k| */
    double max_im;    /* max_k |Im Q_k| (exact path only; 0 on the fast path) */
    double q_norm2;   /* sum_k (Re Q_k)^2 */
    double nyq_bound; /* rigorous bound on ||dropped Nyquist term||_2 / ||Q||_2 (fast path) */
    uint32_t flags;   /* HK_CELL_* bits */
    uint32_t reserved;
    double loss_norm2; /* sum_k (jac f_k L_k)^2, the loss term's scale (fast path; the guard's round-off floor) */
} hk_cell_status;

#define HK_CELL_EXACT 1u            /* evaluated on the exact (full complex) path */
#define HK_CELL_RESIDUE 2u          /* max|Im| > 1e-10 max|Re| (reference would throw, src/spectral.cpp:150) */
#define HK_CELL_GUARD_REROUTED 4u   /* listed by the Nyquist guard; its exact Nyquist term was added (hk_nyqfix) */

/* hk_collision_batch flags */
#define HK_COLL_EXACT 1u  /* every cell on the exact path (complex ga, gb per direction) */
#define HK_COLL_STRICT 2u /* exact + reference throw semantics: HK_NUMERICAL_CONSISTENCY, lowest cell */
#define HK_COLL_NOGUARD 4u /* fast path without the Nyquist guard (benchmark/diagnostic only) */

typedef struct hk_ctx_s* hk_ctx;
typedef struct hk_kernel_s* hk_kernel;

/* ---- context: one per (host thread, GPU) --------------------------------- */
int hk_ctx_create(int device, hk_ctx* out);
int hk_ctx_destroy(hk_ctx ctx);
/* stream: a cudaStream_t (NULL = legacy default stream). */
int hk_ctx_set_stream(hk_ctx ctx, void* stream);
/* Releases the context's cached device workspaces (collision scratch, IMEX /
 * hybrid step work fields); they are re-allocated on the next call that needs
 * them.  Synchronises the context's stream. */
int hk_ctx_trim(hk_ctx ctx);
/* Last error message and failing cell index (-1 if none). */
int hk_last_error(hk_ctx ctx, int64_t* cell, char* msg, size_t msg_len);
/* Number of this library's kernel launches since context creation. */
int64_t hk_launch_count(hk_ctx ctx);
/* Stream-ordered device memory and copies on the context stream (for callers
 * that hold no CUDA runtime of their own, e.g. the C++ mirror hykin_b200.hpp).
 * hk_copy_to_host synchronises the stream before returning. */
int hk_device_alloc(hk_ctx ctx, size_t bytes, void** out);
int hk_device_free(hk_ctx ctx, void* p);
int hk_copy_to_device(hk_ctx ctx, void* dst_dev, const void* src_host, size_t bytes);
int hk_copy_to_host(hk_ctx ctx, void* dst_host, const void* src_dev, size_t bytes);
int hk_ctx_synchronize(hk_ctx ctx);
/* CUDA-event timing of the library's kernels on the context stream (for the
 * roofline in bench.py).  Enabling clears previous records.  tag 0 = main
 * collision kernel, 1 = Nyquist guard, 2 = Nyquist correction of the listed
 * cells; PR(2,2,2) steps: 10 = stage 1, 11 = transport of Y1, 12 = stage 2
 * (f_acc fused), 13 = transport of Y2 (+ final combination). */
int hk_ctx_set_timing(hk_ctx ctx, int on);
int hk_ctx_timing_report(hk_ctx ctx, int tag, double* total_ms, int64_t* launches);

/* ---- spectral kernel ------------------------------------------------------
 * Replaces SpectralKernel precompute_kernel(const VelocityGrid&, int n, int a1,
 * int a2, double r_phys)   (inc/spectral.hpp:49, src/spectral.cpp:53-112).
 * Weight tables are evaluated on the device from the closed forms of the
 * radial/planar transforms (they agree with the GK15 quadrature of
 * src/quadrature.cpp to ~1e-14 relative).  Same validation and status:
 * HK_CONFIG (a1,a2 < 1, n < 2, vmax <= 0, r_phys <= 0), HK_ALIASING
 * (r_phys > 2 vmax/(3+sqrt 2)), HK_UNSUPPORTED (n not in {16, 32, 64}). */
int hk_kernel_create(hk_ctx ctx, int n, int a1, int a2, double vmax, double r_phys,
                     hk_kernel* out);
/* Same, but takes the reference's own tables verbatim (SpectralKernel::alpha,
 * alpha_prime [a1*a2][n^3], loss_diag [n^3], inc/spectral.hpp:25-27). */
int hk_kernel_create_from_tables(hk_ctx ctx, int n, int a1, int a2, double vmax, double r_phys,
                                 const double* alpha_host, const double* alpha_prime_host,
                                 const double* loss_diag_host, hk_kernel* out);
int hk_kernel_destroy(hk_kernel k);
/* out[0..5] = r, jacobian, weight, r_phys, distinct directions, a2 multiplicity of p=0 */
int hk_kernel_info(hk_kernel k, double* out6);

/* ---- collision operator ---------------------------------------------------
 * Replaces void spectral_collision(std::span<const double> f, const
 * SpectralKernel&, std::span<double> out)   (inc/spectral.hpp:56,
 * src/spectral.cpp:114-154), batched over ncells cells.  q_dev receives
 * Re Q per cell.  st_dev (nullable) receives one hk_cell_status per cell.
 * Default: fast path (Hermitian-packed, one complex 3-D transform per
 * direction) with a rigorous per-cell Nyquist guard: any cell whose dropped
 * term could exceed 5e-11 of max(||Q||_2, 2e-5 ||jac f L||_2) gets that term
 * computed exactly and added (Re Q then equals the exact path's).
 * At n = 16 the default is the exact path (a 16^3 spectrum always reaches the
 * Nyquist planes, the guard would list every cell).
 * HK_COLL_EXACT: the reference's arithmetic (two complex transforms per
 * direction) for every cell; HK_COLL_NOGUARD: fast path only.
 * HK_COLL_STRICT returns HK_NUMERICAL_CONSISTENCY (hk_last_error gives the
 * lowest failing cell) when any cell's residue exceeds 1e-10, after writing
 * q_dev for every cell — the reference's throw-after-write behaviour. */
int hk_collision_batch(hk_ctx ctx, hk_kernel k, const double* f_dev, double* q_dev,
                       int64_t ncells, uint32_t flags, hk_cell_status* st_dev);
/* End-to-end variant over host buffers: H2D of f, collision, D2H of q (and
 * st_host if non-NULL), synchronous.  This is the call the reference-facing
 * C++ shim (include/hykin_b200.hpp) makes for spectral_collision. */
int hk_collision_batch_host(hk_ctx ctx, hk_kernel k, const double* f_host, double* q_host,
                            int64_t ncells, uint32_t flags, hk_cell_status* st_host);


/* ---- moments, relaxation stages, classifier, transport ----------------------
 * Per-cell operators over a cell-major slab [ncells][n^3] (device pointers).
 * Per-cell status arrays (int, nullable) receive HK_* codes; the reference
 * would throw the corresponding exception for that cell. */

/* moments_of (src/moments.cpp:21-53) -> mom[cell] = (rho, ux, uy, uz, T);
 * second_moment (:55-81) -> sigma[cell] = (xx, xy, xz, yy, yz, zz);
 * realizability_matrix (:269-312) -> real[cell] = (a_bar 3x3 row-major, b_bar[3], c_bar);
 * l1_distance_to_maxwellian (src/indicators.cpp:89-98) -> l1[cell].  Each output nullable. */
int hk_moments_batch(hk_ctx ctx, int n, double vmax, const double* f_dev, int64_t ncells, double* mom_dev,
                     double* sigma_dev, double* real_dev, double* l1_dev, int* status_dev);
/* maxwellian (src/moments.cpp:88-112) of mom[cell] = (rho, ux, uy, uz, T). */
int hk_maxwellian_batch(hk_ctx ctx, int n, double vmax, const double* mom_dev, int64_t ncells, double* out_dev,
                        int* status_dev);
/* anisotropic_gaussian (src/moments.cpp:120-157, inc/moments.hpp:55): theta[cell] = the
 * stress tensor Theta (3x3 row-major) of mom[cell]; T_c = (1 - beta) T I + beta Theta;
 * fallback[cell] (nullable) = 1 when T_c fails LLT and the Maxwellian was written. */
int hk_anisotropic_gaussian_batch(hk_ctx ctx, int n, double vmax, const double* mom_dev, const double* theta_dev,
                                  double beta, int64_t ncells, double* out_dev, int* fallback_dev);
/* match_moments (src/moments.cpp:225-246, inc/moments.hpp:62), in place:
 * target[cell] = (rho, momentum x, y, z, energy); status HK_DEGENERATE = singular system
 * (the reference throws degenerate_state_error; the cell is left unchanged). */
int hk_match_moments_batch(hk_ctx ctx, int n, double vmax, double* f_dev, const double* target_dev, int64_t ncells,
                           int* status_dev);
/* remove_invariant_moments (src/moments.cpp:248-267, inc/moments.hpp:68), in place on q
 * with weight w and centre uc[cell] (3 doubles); HK_DEGENERATE = singular coupling. */
int hk_remove_invariant_moments_batch(hk_ctx ctx, int n, double vmax, double* q_dev, const double* weight_dev,
                                      const double* uc_dev, int64_t ncells, int* status_dev);
/* esbgk_stage_solve (src/esbgk.cpp:9-45, inc/esbgk.hpp:36): per-cell Knudsen
 * number eps_dev[cell] (or the scalar eps when eps_dev is NULL); nu = nu_coeff rho.
 * info[cell] = status | (gaussian_fallback << 8); mom_dev (nullable) = moments of f*. */
int hk_esbgk_stage_batch(hk_ctx ctx, int n, double vmax, const double* f_star_dev, double* out_dev, int64_t ncells,
                         double a, const double* eps_dev, double eps, double beta, double nu_coeff, int* info_dev,
                         double* mom_dev);
/* penalized_stage_solve (src/boltzmann.cpp:29-45, inc/boltzmann.hpp:36): rate pen_coeff rho. */
int hk_penalized_stage_batch(hk_ctx ctx, int n, double vmax, const double* f_star_dev, double* out_dev,
                             int64_t ncells, double a, const double* eps_dev, double eps, double pen_coeff,
                             int* info_dev, double* mom_dev);
/* penalized_residual (src/boltzmann.cpp:9-27, inc/boltzmann.hpp:29): Q(f) + beta (f - M~),
 * invariant moments projected out.  The collision part follows `flags` as
 * hk_collision_batch (the throw-after-write residue verdict is reported in st_dev). */
int hk_penalized_residual_batch(hk_ctx ctx, hk_kernel k, const double* f_dev, double* out_dev, int64_t ncells,
                                double pen_coeff, uint32_t flags, int* status_dev, hk_cell_status* st_dev);
/* spatial_derivatives + v_eps1_eigenvalues + lambda_b_indicator + regime_update
 * (src/indicators.cpp:14-87, src/regime.cpp:25-52) on a periodic nx x ny grid of
 * kinetic cells, prim = prim_from_moments(mom) (src/coupling.cpp:33-35).
 * r_in/r_out int8 layers {0,1,2}; ind[cell] = (lambda_a, lambda_b, lambda_c, lambda_B)
 * (nullable); l1 may be NULL (HK_CONTRACT where Algorithm 1 needs it). */
int hk_classify(hk_ctx ctx, int nx, int ny, double dx, double dy, const double* mom_dev, const double* eps_dev,
                const double* l1_dev, const int8_t* r_in_dev, int8_t* r_out_dev, double* ind_dev, int* status_dev,
                double eta0, double eta1, double delta0, double mu0, double kappa0, int signed_sum);
/* kinetic_transport_rhs_periodic (src/transport.cpp:51-66): CWENO3 upwind.  x_halo = 0:
 * periodic in x, input [ny][nx][n^3]; x_halo >= 2: input [ny][nx + 2 x_halo][n^3] carries
 * ghost columns (x-slab of a partitioned grid), output [ny][nx][n^3].  Periodic in y. */
int hk_transport_rhs(hk_ctx ctx, int n, double vmax, const double* f_dev, double* out_dev, int nx, int ny,
                     int x_halo, double dx, double dy, double eps_weno);
/* esbgk_imex_step (src/esbgk.cpp:47-99) / penalized_imex_step (src/boltzmann.cpp:47-110):
 * one PR(2,2,2) step of a periodic all-kinetic field, in place.  work_dev: 6 nx ny n^3
 * doubles (3 suffice for n a power of two >= 8 with ny >= 3: the regrouped step keeps
 * Y, f_acc and the residual only) or NULL (context-owned, grow-only). */
int hk_esbgk_imex_step(hk_ctx ctx, int n, double vmax, double* f_dev, int nx, int ny, double dx, double dy, double dt,
                       const double* eps_dev, double beta, double nu_coeff, double eps_weno, double* work_dev);
int hk_penalized_imex_step(hk_ctx ctx, hk_kernel k, double* f_dev, int nx, int ny, double dx, double dy, double dt,
                           const double* eps_dev, double pen_coeff, double eps_weno, uint32_t flags,
                           double* work_dev);
/* PR(2,2,2) steps of one x-slab [ny][nx_local][n^3] of a periodic grid split over
 * the ranks of the context's communicator (hk_ctx_comm_init; without one, or with one
 * rank, the slab is its own periodic neighbour): before each transport the two edge
 * columns of the stage field travel to / from the x-neighbours over NCCL on a
 * separate stream, overlapped with that stage's residual (collision), and the
 * transport reads them from halo buffers (the reference's in-process neighbour
 * reads of src/transport.cpp:51-66 across ranks).  Same arithmetic as the periodic
 * steps above otherwise; work_dev: as for the periodic steps (6, or 3, nx_local ny n^3 doubles) or NULL. */
int hk_penalized_imex_step_slab(hk_ctx ctx, hk_kernel k, double* f_dev, int nx_local, int ny, double dx, double dy,
                                double dt, const double* eps_dev, double pen_coeff, double eps_weno, uint32_t flags,
                                double* work_dev);
int hk_esbgk_imex_step_slab(hk_ctx ctx, int n, double vmax, double* f_dev, int nx_local, int ny, double dx, double dy,
                            double dt, const double* eps_dev, double beta, double nu_coeff, double eps_weno,
                            double* work_dev);
/* Transport of an x-slab [ny][nx][n^3] whose two ghost columns per side come from
 * separate buffers left/right [ny][2][n^3] (filled by the NCCL halo exchange). */
int hk_transport_rhs_slab(hk_ctx ctx, int n, double vmax, const double* f_dev, const double* left_dev,
                          const double* right_dev, double* out_dev, int nx, int ny, double dx, double dy,
                          double eps_weno);
/* Fused PR(2,2,2) combinations of src/boltzmann.cpp:60-109 (per-cell eps):
 * op 0: out = (y - f)/a11;  op 1: out = tr + res/eps (res nullable);
 * op 2: out = f + dt q1 + a21 k1;  op 3 (final, in place on out = f):
 * f += dt (w q1 + w (tr + res/eps)) + w k1 + w (y - f_acc)/a22. */
int hk_imex_combine(hk_ctx ctx, int op, int64_t count, int64_t nb, double dt, const double* eps_dev, double* out_dev,
                    const double* f_dev, const double* y_dev, const double* q1_dev, const double* k1_dev,
                    const double* tr_dev, const double* res_dev);
/* out = x + a y + b z (y, z nullable): the partitioner's halo-free elementwise updates. */
int hk_axpby(hk_ctx ctx, int64_t count, double* out_dev, const double* x_dev, double a, const double* y_dev, double b,
             const double* z_dev);

/* ---- Layer 0 (compressible Euler) and layer transitions (SURVEY §8f "next") --
 * Conserved fields are [cell][4] = (rho, rho ux, rho uy, E), cell = j*nx + i,
 * periodic torus, xi = heat ratio.  Bitwise the reference's arithmetic.
 * HK_POSITIVITY (lowest failing cell in hk_last_error) where the reference
 * throws positivity_error; these calls synchronise to report it. */
/* euler_rhs_periodic (src/euler.cpp:159-170): out = -dF/dx - dG/dy (CWENO3 + local LF). */
int hk_euler_rhs_periodic(hk_ctx ctx, const double* u_dev, int nx, int ny, double dx, double dy, double xi,
                          double eps_weno, double* out_dev);
/* tvd_rk2_step_periodic (src/euler.cpp:172-181), in place; work_dev: 8 nx ny doubles or NULL. */
int hk_euler_tvd_rk2_step(hk_ctx ctx, double* u_dev, int nx, int ny, double dx, double dy, double dt, double xi,
                          double eps_weno, double* work_dev);
/* convert_on_transition 0 -> 1 (src/regime.cpp:62-65): f = maxwellian(moments_from_conserved(u)). */
int hk_conserved_to_maxwellian(hk_ctx ctx, int n, double vmax, const double* u_dev, int64_t ncells, double heat_ratio,
                               double* f_dev);
/* convert_on_transition 1 -> 0 (src/regime.cpp:66-70): u = conserved_from_moments(moments_of(f));
 * HK_DEGENERATE as moments_of. */
int hk_distribution_to_conserved(hk_ctx ctx, int n, double vmax, const double* f_dev, int64_t ncells,
                                 double heat_ratio, double* u_dev);
/* Dynamic packing of a regime's cells into a dense batch and back (nb doubles per
 * cell, nb even): dst[k] = src[idx[k]] / dst[idx[k]] = src[k]. */
int hk_gather_cells(hk_ctx ctx, int64_t nb, const double* src_dev, const int64_t* idx_dev, int64_t count,
                    double* dst_dev);
int hk_scatter_cells(hk_ctx ctx, int64_t nb, const double* src_dev, const int64_t* idx_dev, int64_t count,
                     double* dst_dev);

/* ---- embedded obstacles (SURVEY §8f "next" #4) --------------------------------
 * ObstacleSpec (inc/hykin/obstacle.hpp:9-34): geometry in cell indices; shape
 * HK_OBSTACLE_NONE / _RECTANGLE (half extents) / _DISK (radius); the fixed
 * interior state (rho, pressure, ux, uy); a per-step displacement. */
#define HK_OBSTACLE_NONE 0
#define HK_OBSTACLE_RECTANGLE 1
#define HK_OBSTACLE_DISK 2
typedef struct {
    int shape, center_i, center_j, half_i, half_j, radius;
    double rho, pressure, ux, uy;
    int move_di, move_dj;
} hk_obstacle_spec;
/* Cell kinds (enum class CellKind, inc/hykin/grid.hpp:63). */
#define HK_CELL_INTERIOR 0
#define HK_CELL_OBSTACLE 1
#define HK_CELL_FORCED_RING 2
#define HK_CELL_GHOST 3
/* classify_cells (src/grid.cpp:74-110): kind_dev [ny*nx] uint8, cell = j*nx + i;
 * 4-cell ghost frame, footprint, 2-cell forced-kinetic ring.  HK_CONFIG (first
 * offending cell in row-major order in hk_last_error) when the footprint or
 * the ring reaches the ghost frame.  Synchronises. */
int hk_classify_cells(hk_ctx ctx, int64_t nx, int64_t ny, const hk_obstacle_spec* spec, uint8_t* kind_dev);
/* apply_obstacle (src/coupling.cpp:95-147), once per time step.  spec (host)
 * is moved in place; r_dev [cells] int8 regimes, kind_dev [cells] the previous
 * classification (updated), hydro_dev [cells][4] conserved states, f_dev
 * [cells][n^3] the dense distribution field: blocks of newly covered cells are
 * left untouched (the reference releases them), vacated cells get the fixed
 * state's Maxwellian, ring cells leaving layer 0 the Maxwellian of their hydro
 * state.  covered/vacated (nullable host ints) count the transitions.
 * Errors follow the reference's throw points: HK_CONFIG (static obstacle
 * touching the ghost frame) and HK_SCENARIO_END (moving one leaving the
 * domain) before any cell is touched; HK_POSITIVITY / HK_DEGENERATE at the
 * first failing cell, earlier cells updated as the reference's loop leaves
 * them.  Synchronises (one 16-byte read-back). */
int hk_apply_obstacle(hk_ctx ctx, int n, double vmax, hk_obstacle_spec* spec, int64_t nx, int64_t ny, int8_t* r_dev,
                      uint8_t* kind_dev, double* hydro_dev, double* f_dev, double heat_ratio, int* covered,
                      int* vacated);

/* ---- cross-layer stencil synthesis (src/coupling.cpp:57-93; SURVEY §8f "next" #1) --
 * What a stencil at a cell sees in the hybrid field: ghost cells read the
 * closest interior cell (src/grid.cpp:12-16); obstacle cells the fixed state of
 * spec (required when any kind is HK_CELL_OBSTACLE, else nullable); layer-0
 * cells (r == 0) their conserved state; kinetic cells their moments / stored
 * block.  Grids carry the reference's 4-cell ghost frame (nx, ny >= 9).
 * Both calls synchronise once to report the reference's exception. */
/* synthesize_hydro_state for every cell: out_dev [cells][4].  HK_DEGENERATE
 * (lowest cell) when moments_of of a referenced kinetic block throws. */
int hk_synthesize_hydro(hk_ctx ctx, int n, double vmax, int64_t nx, int64_t ny, const hk_obstacle_spec* spec,
                        const int8_t* r_dev, const uint8_t* kind_dev, const double* hydro_dev, const double* f_dev,
                        double heat_ratio, double* out_dev);
/* synthesize_distribution.  List mode (idx_dev != NULL): out_dev[k] = the block
 * seen at cell idx_dev[k], k < count.  Stencil mode (idx_dev == NULL, count and
 * out_dev ignored): in place in the dense field f_dev, every cell that is not
 * kinetic (ghost, obstacle or layer 0) but lies on the transport stencil
 * (+-2 cells along x or y) of a kinetic interior cell gets the synthesized
 * block, so a kinetic transport sweep over f_dev reads exactly the reference's
 * neighbours; *filled (nullable) = blocks written.  HK_POSITIVITY /
 * HK_DEGENERATE (lowest list entry / cell, nothing written) as the reference. */
int hk_synthesize_distributions(hk_ctx ctx, int n, double vmax, int64_t nx, int64_t ny, const hk_obstacle_spec* spec,
                                const int8_t* r_dev, const uint8_t* kind_dev, const double* hydro_dev, double* f_dev,
                                double heat_ratio, const int64_t* idx_dev, int64_t count, double* out_dev,
                                int64_t* filled);

/* ---- hybrid time step (SURVEY §8f "next" #1: the Algorithm-1 driver) --------
 * The reference ships the per-cell pieces (regime_update src/regime.cpp:25-52,
 * convert_on_transition :54-72, synthesize_* src/coupling.cpp:57-93) but not
 * the step driver (simulation.cpp is absent; SPEC.md harness run_scenario,
 * PAPER.md Algorithm 1 and its stencil-synthesis paragraphs).  The step below
 * is the restatement of that loop the oracle (hko_hybrid_step) pins, on a
 * periodic nx x ny torus without obstacles (BASELINE config 4):
 *   1. indicator pass at t^n: hydro view = U (layer 0) or moments_of(f)
 *      (kinetic), L1 distance of the kinetic cells, regime_update per cell
 *      (skipped when update_regimes == 0: the given r is kept);
 *   2. convert_on_transition: 0->1 f = maxwellian(U); 1->0 U = moments(f);
 *   3. layer 0: TVD-RK2 of the hydro view on the whole torus (kinetic cells
 *      enter the Euler stencil through their moments), kept on r == 0 cells;
 *   4. layers 1 and 2: one PR(2,2,2) step of the kinetic cells (ES-BGK stage
 *      solves on r == 1, penalized stage solves + penalized residual on
 *      r == 2), the transport stencil reading the Maxwellian of the t^n hydro
 *      state on the layer-0 cells within +-2 cells of a kinetic cell (frozen
 *      over the step).
 * r_dev [cells] int8 (in/out), hydro_dev [cells][4] conserved (authoritative
 * on layer 0), f_dev [cells][n^3] dense (authoritative on kinetic cells; the
 * layer-0 halo blocks are overwritten), eps_dev [cells].  counts (host,
 * nullable, 6 entries): cells in layers 0/1/2 after the step, transitions
 * 0->1 and 1->0, halo blocks synthesized.  Errors: HK_POSITIVITY /
 * HK_DEGENERATE with the lowest failing cell.  Synchronises 2-3 times. */
typedef struct {
    double eta0, eta1, delta0;  /* Thresholds (inc/indicators.hpp:49-55) */
    double mu0, kappa0;         /* mu = mu0 sqrt(T), kappa = kappa0 sqrt(T) */
    int signed_sum;             /* LaplacianNorm::signed_sum */
    int update_regimes;         /* 1: Algorithm 1 each step; 0: r_dev kept */
    double heat_ratio;          /* 5/3 */
    double esbgk_beta;          /* -1/2 (Pr = 2/3) */
    double nu_coeff;            /* ES-BGK nu = nu_coeff rho (pi/2) */
    double pen_coeff;           /* penalization beta = pen_coeff rho (2 pi) */
    double eps_weno;            /* 1e-6 */
    uint32_t coll_flags;        /* hk_collision_batch flags of the residuals */
    int ghost_x;                /* x-slab use: columns i < ghost_x and i >= nx - ghost_x are exchanged
                                   ghosts whose results are discarded; their residuals are only evaluated
                                   where an interior cell depends on them (0: plain torus) */
    /* Optional residual hook (NULL: evaluated here).  Called twice per step, at Y1
     * and Y2, ALWAYS (also with m2 = 0 and null pointers, so that ranks that balance
     * the work collectively stay in step): y_dev [m2][n^3] are the stage values of
     * the layer-2 cells whose residual the step needs, in batch order; the hook
     * writes penalized_residual(y) (src/boltzmann.cpp:9-27) to res_dev [m2][n^3]
     * and a status per cell to status_dev [m2] (HK_OK or the HK_* code), with
     * every device operation ordered on `stream` (the context's), and returns
     * HK_OK or an error code.  partition.hybrid_step_slab uses it to spread the
     * layer-2 cells of all x-slabs evenly over the ranks (dynamic load balancing). */
    int (*residual_fn)(void* user, const double* y_dev, double* res_dev, int64_t m2, int* status_dev,
                       void* stream);
    void* residual_user;
} hk_hybrid_params;
int hk_hybrid_step(hk_ctx ctx, hk_kernel k, int nx, int ny, double dx, double dy, double dt, const double* eps_dev,
                   int8_t* r_dev, double* hydro_dev, double* f_dev, const hk_hybrid_params* params, int64_t* counts);
/* hk_hybrid_step on one x-slab of a grid split over the ranks of the context's
 * communicator (hk_ctx_comm_init; without one the slab is its own periodic
 * neighbour): fields [ny][nx_local] (cell j nx_local + i), in place.  One
 * exchange of `ghost` columns of (r, eps, hydro, f) per side (NCCL send/recv
 * into a padded copy), the step on the padded local torus with ghost_x = ghost,
 * the interior copied back: with ghost >= 7 (the step's x-dependency radius)
 * the interior equals the global step's.  counts (nullable) receives the
 * global layer counts [n0, n1, n2] after the step (all-reduced).  The host
 * logic of partition.hybrid_step_slab, in C++. */
int hk_hybrid_step_slab(hk_ctx ctx, hk_kernel k, int nx_local, int ny, double dx, double dy, double dt,
                        const double* eps_dev, int8_t* r_dev, double* hydro_dev, double* f_dev,
                        const hk_hybrid_params* params, int ghost, int64_t* counts);

/* write_snapshot (src/snapshot.cpp is listed by the reference's
 * CMake but not shipped): in directory `dir`, moments_<step>.csv (i,j,x,y,rho,ux,uy,T,P,
 * one row per cell, c = j nx + i, cell centres), regimes_<step>.txt (ny lines of nx
 * layers; -1 where kind_dev marks HK_CELL_OBSTACLE, kind_dev nullable) and
 * meta_<step>.json (step, time, grids, heat ratio, config_json echoed verbatim or
 * null).  Layer-0 cells: prim_from_conserved of hydro_dev; kinetic cells:
 * prim_from_moments of moments_of(f_dev).  HK_POSITIVITY / HK_DEGENERATE with the
 * lowest non-physical cell, HK_IO (io_error) when the files cannot be written. */
int hk_write_snapshot(hk_ctx ctx, int n, double vmax, int64_t nx, int64_t ny, double dx, double dy,
                      const int8_t* r_dev, const uint8_t* kind_dev, const double* hydro_dev, const double* f_dev,
                      double heat_ratio, int64_t step, double time, const char* dir, const char* config_json);

/* ---- multi-GPU: NCCL communicator of a context ------------
 * One process per GPU.  Rank 0 calls hk_comm_unique_id, the host side ships
 * the 128 opaque bytes to every rank (MPI / torch.distributed / a file), and
 * each rank calls hk_ctx_comm_init on its context.  NCCL is loaded at run
 * time (libnccl.so.2); HK_NCCL if it is absent or a collective fails. */
#define HK_COMM_ID_BYTES 128
int hk_comm_unique_id(void* id_out /* HK_COMM_ID_BYTES */);
int hk_ctx_comm_init(hk_ctx ctx, int nranks, int rank, const void* id /* HK_COMM_ID_BYTES */);
int hk_ctx_comm_info(hk_ctx ctx, int* nranks, int* rank);
/* x-slab halo exchange before a transport sweep (kinetic_transport_rhs_periodic's
 * neighbour reads, src/transport.cpp:51-66, across ranks).  f: [ny][nx_local][n^3];
 * left <- last two columns of rank-1, right <- first two columns of rank+1
 * (periodic over ranks), each [ny][2][n^3] — the layout hk_transport_rhs_slab reads. */
int hk_halo_exchange(hk_ctx ctx, int n, const double* f_dev, int64_t nx_local, int64_t ny, double* left_dev,
                     double* right_dev);
/* Halo-free variant over NVLink / NVSwitch peer memory: the transport kernel
 * reads the two ghost columns straight from the neighbour ranks' slabs
 * ([ny][left_nx][n^3], last two columns; [ny][right_nx][n^3], first two),
 * mapped into this process with hk_ipc_open.  No exchange step; the caller
 * orders the neighbours' writes before the call (stream sync + barrier). */
int hk_transport_rhs_peer(hk_ctx ctx, int n, double vmax, const double* f_dev, const double* left_slab_dev,
                          int left_nx, const double* right_slab_dev, int right_nx, double* out_dev, int nx, int ny,
                          double dx, double dy, double eps_weno);
/* CUDA IPC of a device buffer (64-byte handle): export on the owner, open on a
 * peer; the opened pointer is the allocation base, add *offset_out (nullable). */
#define HK_IPC_HANDLE_BYTES 64
int hk_ipc_handle(hk_ctx ctx, const void* dev_ptr, void* handle_out /* HK_IPC_HANDLE_BYTES */, int64_t* offset_out);
int hk_ipc_open(hk_ctx ctx, const void* handle, void** dev_ptr_out);
int hk_ipc_close(hk_ctx ctx, void* dev_ptr);
/* In-place all-reduce of `count` doubles over the context's ranks: regime counts,
 * conservation sums (HK_REDUCE_SUM), CFL / residual maxima (HK_REDUCE_MAX). */
#define HK_REDUCE_SUM 0
#define HK_REDUCE_MAX 1
int hk_allreduce_scalars(hk_ctx ctx, double* buf_dev, int64_t count, int op);

/* ---- diagnostics ---------------------------------------------------------- */
/* fp64 FMA peak of this device (DFMA microbenchmark), TFLOP/s. */
double hk_measure_fp64_peak(hk_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif
