/*
 * hk_oracle.h — CPU restatement of the hykin fast-spectral collision path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the CPU baseline.  The product path (paper_2505_03360_b200/) never links it.
 *
 * Every function restates one reference function; the citation is given as
 * file:line relative to /root/reference/proj/core (src/ = sources,
 * inc/ = include/hykin).  Loop nests and summation orders follow the
 * reference so that results agree to round-off.
 *
 * Parity pin: this restatement is checked against the reference's own
 * sources compiled here (oracle/_ref, see oracle/Makefile) and against the
 * golden vectors those produced (tests/golden/).  FFTW3 and Eigen3 are absent
 * from this image; both builds use the same radix-2 FFT (hko_fft_1d) and the
 * Eigen-subset shim, so the pin covers the reference's arithmetic with a
 * stand-in FFT / dense-LA library.
 *
 * Layouts: a velocity block is n^3 doubles, index (k1*n + k2)*n + k3
 * (inc/grid.hpp:54).  Complex arrays are interleaved (re, im).  Fields are
 * contiguous cell-major slabs [cell][k1][k2][k3], cell = j*nx + i
 * (inc/grid.hpp:30).
 */
#ifndef HK_ORACLE_H
#define HK_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes mirror inc/errors.hpp:9-61 (same values as include/hykin_b200.h). */
enum {
    HKO_OK = 0,
    HKO_CONFIG = 1,                /* config_error */
    HKO_ALIASING = 2,              /* aliasing_config_error */
    HKO_DEGENERATE = 3,            /* degenerate_state_error */
    HKO_NUMERICAL_CONSISTENCY = 4, /* numerical_consistency_error */
    HKO_CONTRACT = 5,              /* contract_violation */
    HKO_POSITIVITY = 8,            /* positivity_error */
    HKO_SCENARIO_END = 10          /* scenario_end_error */
};

/* ---------------- FFT (stand-in for FFTW3 C2C, src/fft.cpp:35-40) ---------------- */
/* In-place complex DFT of length n with stride (in complex elements).
 * sign = -1: X_k = sum_j x_j e^{-2 pi i jk/n} (FFTW_FORWARD); +1 backward.
 * Unnormalised, like FFTW.  Radix-2 for powers of two, direct DFT otherwise. */
void hko_fft_1d(int n, double* data, long stride, int sign);
/* 3-D row-major n^3 complex transform, unnormalised (fftw_plan_dft_3d). */
void hko_fft_3d(int n, double* data, int sign);
/* 2-D row-major n^2 complex transform, unnormalised (fftw_plan_dft_2d). */
void hko_fft_2d(int n, double* data, int sign);
/* Accurate e^{i 2 pi k / n} via octant reduction. */
void hko_unit_root(long k, long n, double* c, double* s);

/* ---------------- grid (src/grid.cpp:18-33) ---------------- */
double hko_node(int n, double vmax, int k);
double hko_dv(int n, double vmax);
double hko_dvk(int n, double vmax);

/* ---------------- quadrature (src/quadrature.cpp:11-63) ---------------- */
double hko_gk15_radial(double s, double r, double amp);  /* src/spectral.cpp:43-46 */
double hko_gk15_planar(double s, double r, double amp);  /* src/spectral.cpp:48-51 */
/* Closed forms of the two transforms. */
double hko_closed_radial(double s, double r, double amp);
double hko_closed_planar(double s, double r, double amp);

/* ---------------- spectral kernel (src/spectral.cpp:53-112) ---------------- */
typedef struct {
    int n, a1, a2;
    double vmax, r_phys, r, jacobian, weight;
    double* alpha;       /* [a1*a2][n^3] */
    double* alpha_prime; /* [a1*a2][n^3] */
    double* loss_diag;   /* [n^3] */
} hko_kernel;

/* closed_form = 0 restates the adaptive GK15 quadrature exactly; 1 uses the
 * closed forms (agree to ~3e-13 of phi(0)).  nthreads > 1 splits directions. */
int hko_precompute(int n, double vmax, int a1, int a2, double r_phys, int closed_form,
                   int nthreads, hko_kernel* k);
void hko_kernel_free(hko_kernel* k);

/* src/spectral.cpp:114-154.  Writes out = Re Q, then returns
 * HKO_NUMERICAL_CONSISTENCY if max|Im Q| > 1e-10 max|Re Q| (the reference
 * throws after writing out).  residue (nullable) = max|Im| / max(max|Re|,1e-300).
 * gain_out / loss_out (nullable, complex n^3) expose the intermediates. */
int hko_spectral_collision(const hko_kernel* k, const double* f, double* out, double* residue);

/* Batch over cells with a WorkerPool-style contiguous partition
 * (inc/threading.hpp:25-56).  Per-cell statuses / residues into st / res. */
int hko_collision_batch(const hko_kernel* k, const double* f, double* q, long ncells,
                        int nthreads, int* st, double* res);

/* ---------------- moments (src/moments.cpp) ---------------- */
typedef struct {
    double rho, u[3], T;
} hko_moments;

int hko_moments_of(int n, double vmax, const double* f, hko_moments* m);          /* :21-53 */
void hko_second_moment(int n, double vmax, const double* f, double s[9]);         /* :55-81 */
void hko_stress_tensor(int n, double vmax, const double* f, const hko_moments* m,
                       double theta[9]);                                          /* :83-86 */
int hko_maxwellian(const hko_moments* m, int n, double vmax, double* out);        /* :88-112 */
int hko_anisotropic_gaussian(const hko_moments* m, const double theta[9], double beta,
                             int n, double vmax, double* out, int* fell_back);    /* :120-157 */
int hko_match_moments(double* f, int n, double vmax, double rho, const double mom[3],
                      double energy);                                            /* :225-246 */
int hko_remove_invariant_moments(double* q, const double* weight, int n, double vmax,
                                 const double uc[3]);                            /* :248-267 */
void hko_realizability_matrix(const double* f, int n, double vmax, const hko_moments* m,
                              double a_bar[9], double b_bar[3], double* c_bar);   /* :269-312 */
void hko_realizability_5x5(const double a_bar[9], const double b_bar[3], double c_bar,
                           double m[25]);                                         /* :9-19 */
/* Full-pivot LU solve with Eigen's FullPivLU invertibility threshold. */
int hko_solve5(const double a[25], const double rhs[5], double x[5]);

/* ---------------- Boltzmann layer (src/boltzmann.cpp) ---------------- */
int hko_penalized_residual(const hko_kernel* k, const double* f, double pen_coeff,
                           double* out, double* residue);                        /* :9-27 */
int hko_penalized_stage_solve(const double* f_star, double a, double eps, double pen_coeff,
                              int n, double vmax, double* out, hko_moments* m);  /* :29-45 */
int hko_penalized_imex_step(double* f, int nx, int ny, const hko_kernel* k, double dx,
                            double dy, double dt, const double* eps_cell, double pen_coeff,
                            double eps_weno, int nthreads);                       /* :47-110 */

/* ---------------- ES-BGK layer (src/esbgk.cpp) ---------------- */
int hko_esbgk_stage_solve(const double* f_star, double a, double eps, double beta,
                          double nu_coeff, int n, double vmax, double* out, hko_moments* m,
                          int* fallback);                                        /* :9-45 */
int hko_esbgk_imex_step(double* f, int nx, int ny, int n, double vmax, double dx, double dy,
                        double dt, const double* eps_cell, double beta, double nu_coeff,
                        double eps_weno, int nthreads);                           /* :47-99 */

/* ---------------- indicators + regime (src/indicators.cpp, src/regime.cpp) ---------------- */
/* prim = (rho, ux, uy, T).  d[11] = drho_dx, drho_dy, dux_dx, dux_dy, duy_dx, duy_dy,
 * dT_dx, dT_dy, lap_rho, lap_ux, lap_uy  (inc/indicators.hpp:19-27). */
void hko_spatial_derivatives(const double c[4], const double xm[4], const double xp[4],
                             const double ym[4], const double yp[4], double dx, double dy,
                             double d[11]);                                       /* :14-32 */
void hko_v_eps1_eigenvalues(const double d[11], const double prim[4], double eps, double mu0,
                            double kappa0, double lam[3]);                        /* :60-73 */
double hko_lambda_b(const double d[11], const double prim[4], double eps, int signed_sum);/* :75-87 */
int hko_l1_distance(const double* f, int n, double vmax, double* out);           /* :89-98 */
/* src/regime.cpp:25-52.  lam / lambda_b / l1 nullable (= indicator absent). */
int hko_regime_update(int r, const double* lam, const double* lambda_b, const double* l1,
                      double eta0, double eta1, double delta0, int* out);

/* ---------------- transport (src/transport.cpp, src/euler.cpp:10-40) ---------------- */
void hko_cweno3(double um, double uc, double up, double eps, double* left, double* right);
void hko_transport_rhs_cell(const double* const fx[5], const double* const fy[5], int n,
                            double vmax, double dx, double dy, double eps_weno, double* out);
void hko_transport_rhs_periodic(const double* f, int nx, int ny, int n, double vmax, double dx,
                                double dy, double eps_weno, double* out);

/* ---------------- Layer-0 Euler (src/euler.cpp:67-189) ---------------- */
/* u, out: [cell][4] = (rho, mx, my, E), cell = j*nx + i, periodic torus.
 * Returns HKO_POSITIVITY (and *bad_cell) on a non-positive density / pressure
 * of a cell state or of a reconstructed face state, as the reference throws. */
int hko_euler_rhs_periodic(const double* u, int nx, int ny, double dx, double dy, double xi,
                           double eps_weno, double* out, long* bad_cell);        /* :159-170 */
int hko_tvd_rk2_step_periodic(double* u, int nx, int ny, double dx, double dy, double dt,
                              double xi, double eps_weno, long* bad_cell);      /* :172-181 */
/* Transitions (src/coupling.cpp:7-22, src/regime.cpp:54-72) */
int hko_moments_from_conserved(const double u[4], double heat_ratio, double mom5[5]);
void hko_conserved_from_moments(const double mom5[5], double heat_ratio, double u[4]);

/* ---------------- obstacles (src/grid.cpp:56-110, src/coupling.cpp:95-147) ---------------- */
typedef struct {
    int shape; /* 0 none, 1 rectangle, 2 disk (ObstacleSpec::Shape) */
    int center_i, center_j, half_i, half_j, radius;
    double rho, pressure, ux, uy;
    int move_di, move_dj;
} hko_obstacle;
/* kind: 0 interior, 1 obstacle, 2 forced_ring, 3 ghost (CellKind); ghost frame depth 4. */
int hko_classify_cells(int nx, int ny, const hko_obstacle* s, unsigned char* kind, long* bad_cell);
/* Dense f [cells][n^3]: released (covered) blocks are left untouched. Returns
 * HKO_CONFIG / HKO_SCENARIO_END / HKO_POSITIVITY like the reference throws. */
int hko_apply_obstacle(int nx, int ny, int n, double vmax, hko_obstacle* s, signed char* r, unsigned char* kind,
                       double* hydro, double* f, double heat_ratio, int* covered, int* vacated);
/* Cross-layer stencil synthesis (src/coupling.cpp:57-93) at cell (i, j) of an
 * nx x ny grid: ghost cells read their clamped interior cell (src/grid.cpp:12-16).
 * hydro [cells][4], f dense [cells][n^3]; s may be NULL when no cell is an obstacle. */
int hko_synthesize_hydro_state(int nx, int ny, int n, double vmax, const hko_obstacle* s, const signed char* r,
                               const unsigned char* kind, const double* hydro, const double* f, double heat_ratio,
                               int i, int j, double out[4]);
int hko_synthesize_distribution(int nx, int ny, int n, double vmax, const hko_obstacle* s, const signed char* r,
                                const unsigned char* kind, const double* hydro, const double* f, double heat_ratio,
                                int i, int j, double* out);

/* ---------------- hybrid time step (restatement; the reference's driver is absent) ----------------
 * One step of the hybrid scheme on a periodic nx x ny torus without obstacles,
 * as SPEC.md harness run_scenario and PAPER.md Algorithm 1 describe it and as
 * include/hykin_b200.h:hk_hybrid_step states it: indicator pass at t^n
 * (hydro view = U on layer 0, moments_of(f) on kinetic cells), regime_update
 * (src/regime.cpp:25-52), convert_on_transition (:54-72), layer 0 = TVD-RK2
 * of the hydro view (src/euler.cpp:172-181) kept on r == 0, kinetic cells = one
 * PR(2,2,2) step (ES-BGK on r == 1, penalized Boltzmann on r == 2) whose
 * transport stencil reads the frozen Maxwellian of the t^n hydro state on the
 * layer-0 cells within +-2 cells (synthesize_distribution, src/coupling.cpp:72-93).
 * counts (nullable): n0, n1, n2 after the step, transitions 0->1, 1->0, halo
 * blocks.  Returns the first failure (HKO_POSITIVITY / HKO_DEGENERATE). */
typedef struct {
    double eta0, eta1, delta0, mu0, kappa0;
    int signed_sum, update_regimes;
    double heat_ratio, esbgk_beta, nu_coeff, pen_coeff, eps_weno;
} hko_hybrid_params;
int hko_hybrid_step(int nx, int ny, const hko_kernel* k, double dx, double dy, double dt, const double* eps,
                    signed char* r, double* hydro, double* f, const hko_hybrid_params* p, long counts[6]);

#ifdef __cplusplus
}
#endif
#endif
