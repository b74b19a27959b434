/*
 * hk_oracle.c — CPU restatement of the hykin fast-spectral collision path.
 * TEST INFRASTRUCTURE ONLY (see hk_oracle.h).  Citations are relative to
 * /root/reference/proj/core.  Compiled with -O2 -std=c11 and no -march so
 * that no FMA contraction changes the reference's rounding.
 */
#include "hk_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
#ifndef M_SQRT1_2
#define M_SQRT1_2 0.70710678118654752440
#endif

/* ===================================================================== */
/* FFT: stand-in for FFTW3's unnormalised C2C transforms (src/fft.cpp).   */
/* ===================================================================== */

void hko_unit_root(long k, long n, double* c, double* s) {
    /* e^{i 2 pi k/n} with the angle reduced to [0, pi/4] so that the
     * libm call sees a small, exactly-representable-ratio argument. */
    k %= n;
    if (k < 0) k += n;
    long k8 = 8 * k; /* angle = (k8 / n) * (pi/4) */
    long oct = k8 / n;
    long rem = k8 - oct * n; /* angle within octant: rem/n * pi/4 */
    double t = (M_PI / 4.0) * ((double)rem / (double)n);
    double ct = cos(t), st = sin(t);
    double cc, ss;
    /* angle = oct*pi/4 + t */
    switch (oct) {
    case 0: cc = ct; ss = st; break;
    case 1: { double u = M_PI / 4.0 - t; /* angle = pi/2 - u */
              cc = sin(u); ss = cos(u);
              if (rem == 0) { cc = M_SQRT1_2; ss = M_SQRT1_2; } break; }
    case 2: cc = -st; ss = ct; break;
    case 3: { double u = M_PI / 4.0 - t; cc = -cos(u); ss = sin(u);
              if (rem == 0) { cc = -M_SQRT1_2; ss = M_SQRT1_2; } break; }
    case 4: cc = -ct; ss = -st; break;
    case 5: { double u = M_PI / 4.0 - t; cc = -sin(u); ss = -cos(u);
              if (rem == 0) { cc = -M_SQRT1_2; ss = -M_SQRT1_2; } break; }
    case 6: cc = st; ss = -ct; break;
    default: { double u = M_PI / 4.0 - t; cc = cos(u); ss = -sin(u);
               if (rem == 0) { cc = M_SQRT1_2; ss = -M_SQRT1_2; } break; }
    }
    *c = cc;
    *s = ss;
}

static int is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

/* Twiddle tables e^{i 2 pi k/n}, k < n, one per power-of-two n, built once
 * (same hko_unit_root values the per-call tables had) and read-only after. */
static double* g_tw[31];
static pthread_mutex_t g_tw_mu = PTHREAD_MUTEX_INITIALIZER;

static const double* twiddles(int n) {
    int lg = 0;
    while ((1 << lg) < n) ++lg;
    double* t = __atomic_load_n(&g_tw[lg], __ATOMIC_ACQUIRE);
    if (t) return t;
    pthread_mutex_lock(&g_tw_mu);
    t = g_tw[lg];
    if (!t) {
        t = (double*)malloc(sizeof(double) * 2 * (size_t)n);
        for (int k = 0; k < n; ++k) hko_unit_root(k, n, &t[2 * k], &t[2 * k + 1]);
        __atomic_store_n(&g_tw[lg], t, __ATOMIC_RELEASE);
    }
    pthread_mutex_unlock(&g_tw_mu);
    return t;
}

/* Radix-2 DIT over B pencils at once: x is [n][B] complex (pencil b of row j
 * at x[2*(j*B+b)]).  Every pencil sees exactly the butterfly sequence of the
 * single-pencil transform (bit reversal, then len = 2, 4, ..., n), so the
 * results are bitwise those of B separate 1-D transforms. */
static void fft_pow2_multi(int n, int B, double* x, int sign, const double* tw) {
    for (int i = 1, j = 0; i < n; ++i) {
        int bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            double* a = x + 2 * (size_t)i * B;
            double* b = x + 2 * (size_t)j * B;
            for (int q = 0; q < 2 * B; ++q) { double t = a[q]; a[q] = b[q]; b[q] = t; }
        }
    }
    for (int len = 2; len <= n; len <<= 1) {
        int half = len >> 1, step = n / len;
        for (int i = 0; i < n; i += len) {
            for (int j = 0; j < half; ++j) {
                const double wr = tw[2 * (j * step)], wi = sign * tw[2 * (j * step) + 1];
                double* a = x + 2 * (size_t)(i + j) * B;
                double* b = x + 2 * (size_t)(i + j + half) * B;
                for (int q = 0; q < B; ++q) {
                    double br = b[2 * q] * wr - b[2 * q + 1] * wi;
                    double bi = b[2 * q] * wi + b[2 * q + 1] * wr;
                    b[2 * q] = a[2 * q] - br; b[2 * q + 1] = a[2 * q + 1] - bi;
                    a[2 * q] = a[2 * q] + br; a[2 * q + 1] = a[2 * q + 1] + bi;
                }
            }
        }
    }
}

static void dft_naive(int n, double* data, long stride, int sign, const double* tw, double* buf) {
    for (int j = 0; j < n; ++j) {
        buf[2 * j] = data[2 * j * stride];
        buf[2 * j + 1] = data[2 * j * stride + 1];
    }
    for (int k = 0; k < n; ++k) {
        double sr = 0.0, si = 0.0;
        for (int j = 0; j < n; ++j) {
            long m = ((long)j * k) % n;
            double wr = tw[2 * m], wi = sign * tw[2 * m + 1];
            sr += buf[2 * j] * wr - buf[2 * j + 1] * wi;
            si += buf[2 * j] * wi + buf[2 * j + 1] * wr;
        }
        data[2 * k * stride] = sr;
        data[2 * k * stride + 1] = si;
    }
}

void hko_fft_1d(int n, double* data, long stride, int sign) {
    if (is_pow2(n)) {
        const double* tw = twiddles(n);
        if (stride == 1) {
            fft_pow2_multi(n, 1, data, sign, tw);
            return;
        }
        double* buf = (double*)malloc(sizeof(double) * 2 * (size_t)n);
        for (int j = 0; j < n; ++j) {
            buf[2 * j] = data[2 * j * stride];
            buf[2 * j + 1] = data[2 * j * stride + 1];
        }
        fft_pow2_multi(n, 1, buf, sign, tw);
        for (int j = 0; j < n; ++j) {
            data[2 * j * stride] = buf[2 * j];
            data[2 * j * stride + 1] = buf[2 * j + 1];
        }
        free(buf);
        return;
    }
    double* buf = (double*)malloc(sizeof(double) * 4 * (size_t)n);
    double* tw = buf + 2 * n;
    for (int k = 0; k < n; ++k) hko_unit_root(k, n, &tw[2 * k], &tw[2 * k + 1]);
    dft_naive(n, data, stride, sign, tw, buf);
    free(buf);
}

/* Pencils p0 .. p0+B-1 of a strided axis: pencil p, element j at
 * d[2*(p*pstride + j*stride)] with pstride = 1 (adjacent pencils), gathered
 * into a [n][B] tile, transformed, scattered back. */
static void fft_strided_block(int n, double* d, long stride, int B, double* tile, int sign,
                              const double* tw) {
    for (int j = 0; j < n; ++j)
        memcpy(tile + 2 * (size_t)j * B, d + 2 * (size_t)j * stride, sizeof(double) * 2 * B);
    fft_pow2_multi(n, B, tile, sign, tw);
    for (int j = 0; j < n; ++j)
        memcpy(d + 2 * (size_t)j * stride, tile + 2 * (size_t)j * B, sizeof(double) * 2 * B);
}

#define HKO_FFT_TILE 32  /* pencils per strided tile: 32 x 32 complex = 16 KiB (L1); vectorises over the tile */

void hko_fft_3d(int n, double* d, int sign) {
    const long n2 = (long)n * n;
    if (!is_pow2(n)) {
        for (long p = 0; p < n2; ++p) hko_fft_1d(n, d + 2 * p * n, 1, sign);         /* axis 3 */
        for (int i1 = 0; i1 < n; ++i1)
            for (int i3 = 0; i3 < n; ++i3) hko_fft_1d(n, d + 2 * (i1 * n2 + i3), n, sign); /* axis 2 */
        for (long p = 0; p < n2; ++p) hko_fft_1d(n, d + 2 * p, n2, sign);             /* axis 1 */
        return;
    }
    const double* tw = twiddles(n);
    const int B = n < HKO_FFT_TILE ? n : HKO_FFT_TILE;
    double* tile = (double*)malloc(sizeof(double) * 2 * (size_t)n * B);
    for (long p = 0; p < n2; ++p) fft_pow2_multi(n, 1, d + 2 * p * n, sign, tw); /* axis 3 */
    for (int i1 = 0; i1 < n; ++i1)                                               /* axis 2 */
        for (int i3 = 0; i3 < n; i3 += B) fft_strided_block(n, d + 2 * (i1 * n2 + i3), n, B, tile, sign, tw);
    for (long p = 0; p < n2; p += B) fft_strided_block(n, d + 2 * p, n2, B, tile, sign, tw); /* axis 1 */
    free(tile);
}

void hko_fft_2d(int n, double* d, int sign) {
    if (!is_pow2(n)) {
        for (int i = 0; i < n; ++i) hko_fft_1d(n, d + 2 * (long)i * n, 1, sign);
        for (int j = 0; j < n; ++j) hko_fft_1d(n, d + 2 * j, n, sign);
        return;
    }
    const double* tw = twiddles(n);
    const int B = n < HKO_FFT_TILE ? n : HKO_FFT_TILE;
    double* tile = (double*)malloc(sizeof(double) * 2 * (size_t)n * B);
    for (int i = 0; i < n; ++i) fft_pow2_multi(n, 1, d + 2 * (long)i * n, sign, tw);
    for (int j = 0; j < n; j += B) fft_strided_block(n, d + 2 * j, n, B, tile, sign, tw);
    free(tile);
}

/* ===================================================================== */
/* grid (src/grid.cpp:18-33)                                             */
/* ===================================================================== */

double hko_dv(int n, double vmax) { return 2.0 * vmax / n; }
double hko_dvk(int n, double vmax) {
    const double dv = hko_dv(n, vmax);
    return dv * dv * dv;
}
double hko_node(int n, double vmax, int k) { return -vmax + (k + 0.5) * hko_dv(n, vmax); }

static int fft_frequency(int idx, int n) { return idx < n / 2 ? idx : idx - n; } /* inc/fft.hpp:69 */

/* ===================================================================== */
/* quadrature: adaptive Gauss-Kronrod 7/15 (src/quadrature.cpp:11-63)    */
/* ===================================================================== */

static const double kx[15] = {
    -0.991455371120813, -0.949107912342759, -0.864864423359769, -0.741531185599394,
    -0.586087235467691, -0.405845151377397, -0.207784955007898, 0.0,
    0.207784955007898,  0.405845151377397,  0.586087235467691,  0.741531185599394,
    0.864864423359769,  0.949107912342759,  0.991455371120813};
static const double kw[15] = {
    0.022935322010529, 0.063092092629979, 0.104790010322250, 0.140653259715525,
    0.169004726639267, 0.190350578064785, 0.204432940075298, 0.209482141084728,
    0.204432940075298, 0.190350578064785, 0.169004726639267, 0.140653259715525,
    0.104790010322250, 0.063092092629979, 0.022935322010529};
static const double gw[7] = {0.129484966168870, 0.279705391489277, 0.381830050505119,
                             0.417959183673469, 0.381830050505119, 0.279705391489277,
                             0.129484966168870};

typedef double (*integrand_fn)(double rho, double s);

static double f_radial(double rho, double s) { return rho * cos(rho * s); }
static double sinc_ref(double x) { return x == 0.0 ? 1.0 : sin(x) / x; } /* src/spectral.cpp:16 */
static double f_planar(double rho, double s) { return rho * sinc_ref(rho * s); }

typedef struct { double integral, error; } panel;

static panel gk15(integrand_fn f, double s, double a, double b) {
    const double c = 0.5 * (a + b), h = 0.5 * (b - a);
    double ik = 0.0, ig = 0.0;
    for (int i = 0; i < 15; ++i) {
        const double v = f(c + h * kx[i], s);
        ik += kw[i] * v;
        if (i % 2 == 1) ig += gw[i / 2] * v;
    }
    panel p = {ik * h, fabs((ik - ig) * h)};
    return p;
}

static double integrate_rec(integrand_fn f, double s, double a, double b, panel whole, double tol,
                            int depth) {
    if (whole.error <= tol || depth >= 48) return whole.integral;
    const double c = 0.5 * (a + b);
    const panel left = gk15(f, s, a, c), right = gk15(f, s, c, b);
    return integrate_rec(f, s, a, c, left, 0.5 * tol, depth + 1) +
           integrate_rec(f, s, c, b, right, 0.5 * tol, depth + 1);
}

static double adaptive_integrate(integrand_fn f, double s, double a, double b) {
    /* default tolerances of inc/quadrature.hpp: abs 1e-12, rel 1e-10 */
    const panel whole = gk15(f, s, a, b);
    const double tol = 1e-12 + 1e-10 * fabs(whole.integral);
    return integrate_rec(f, s, a, b, whole, tol, 0);
}

double hko_gk15_radial(double s, double r, double amp) {
    return 2.0 * amp * adaptive_integrate(f_radial, s, 0.0, r);
}
double hko_gk15_planar(double s, double r, double amp) {
    return 4.0 * amp * adaptive_integrate(f_planar, s, 0.0, r);
}

/* Closed forms: 2 amp int_0^r rho cos(rho s) = 2 amp [r sin(rs)/s - 2 sin^2(rs/2)/s^2],
 * 4 amp int_0^r rho sinc(rho s) = 4 amp * 2 sin^2(rs/2)/s^2; limits amp r^2, 2 amp r^2. */
double hko_closed_radial(double s, double r, double amp) {
    if (s == 0.0) return amp * r * r;
    const double h = sin(0.5 * r * s);
    return 2.0 * amp * (r * sin(r * s) / s - 2.0 * h * h / (s * s));
}
double hko_closed_planar(double s, double r, double amp) {
    if (s == 0.0) return 2.0 * amp * r * r;
    const double h = sin(0.5 * r * s);
    return 8.0 * amp * h * h / (s * s);
}

/* ===================================================================== */
/* spectral kernel precompute (src/spectral.cpp:53-112)                  */
/* ===================================================================== */

typedef struct {
    hko_kernel* k;
    int d0, d1, closed;
} pre_job;

static void* precompute_dirs(void* arg) {
    pre_job* job = (pre_job*)arg;
    hko_kernel* k = job->k;
    const int n = k->n;
    const long total = (long)n * n * n;
    for (int d = job->d0; d < job->d1; ++d) {
        const int p = d / k->a2, q = d % k->a2;
        const double theta = p * M_PI / k->a1;
        const double phi = q * M_PI / k->a2;
        const double e0 = sin(theta) * cos(phi), e1 = sin(theta) * sin(phi), e2 = cos(theta);
        double* a = k->alpha + (long)d * total;
        double* ap = k->alpha_prime + (long)d * total;
        long idx = 0;
        for (int i1 = 0; i1 < n; ++i1) {
            const double l1 = fft_frequency(i1, n);
            for (int i2 = 0; i2 < n; ++i2) {
                const double l2 = fft_frequency(i2, n);
                for (int i3 = 0; i3 < n; ++i3, ++idx) {
                    const double l3 = fft_frequency(i3, n);
                    const double ldote = l1 * e0 + l2 * e1 + l3 * e2;
                    const double l2norm = l1 * l1 + l2 * l2 + l3 * l3;
                    double perp2 = l2norm - ldote * ldote;
                    if (perp2 < 0.0) perp2 = 0.0;
                    if (job->closed) {
                        a[idx] = hko_closed_radial(ldote, k->r, 2.0);
                        ap[idx] = hko_closed_planar(sqrt(perp2), k->r, 2.0);
                    } else {
                        a[idx] = hko_gk15_radial(ldote, k->r, 2.0);
                        ap[idx] = hko_gk15_planar(sqrt(perp2), k->r, 2.0);
                    }
                }
            }
        }
    }
    return NULL;
}

int hko_precompute(int n, double vmax, int a1, int a2, double r_phys, int closed_form,
                   int nthreads, hko_kernel* k) {
    memset(k, 0, sizeof(*k));
    if (n < 2 || vmax <= 0.0) return HKO_CONFIG;                       /* src/grid.cpp:19-22 */
    if (a1 < 1 || a2 < 1) return HKO_CONFIG;                           /* src/spectral.cpp:58 */
    const double r_max = 2.0 * vmax / (3.0 + sqrt(2.0));
    if (r_phys > r_max * (1.0 + 1e-12)) return HKO_ALIASING;           /* :60-64 */
    if (r_phys <= 0.0) return HKO_CONFIG;                              /* :65-66 */
    k->n = n; k->a1 = a1; k->a2 = a2; k->vmax = vmax; k->r_phys = r_phys;
    k->r = r_phys * M_PI / vmax;
    const double s = vmax / M_PI;
    k->jacobian = s * s * s * s;
    k->weight = M_PI * M_PI / (a1 * a2);
    const long total = (long)n * n * n;
    const int dirs = a1 * a2;
    k->alpha = (double*)malloc(sizeof(double) * total * dirs);
    k->alpha_prime = (double*)malloc(sizeof(double) * total * dirs);
    k->loss_diag = (double*)calloc((size_t)total, sizeof(double));
    if (nthreads < 1) nthreads = 1;
    if (nthreads > dirs) nthreads = dirs;
    pthread_t th[256];
    pre_job jobs[256];
    if (nthreads > 256) nthreads = 256;
    const int chunk = (dirs + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].k = k;
        jobs[t].d0 = t * chunk;
        jobs[t].d1 = (t + 1) * chunk < dirs ? (t + 1) * chunk : dirs;
        jobs[t].closed = closed_form;
        if (t > 0) pthread_create(&th[t], NULL, precompute_dirs, &jobs[t]);
    }
    precompute_dirs(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    /* loss_diag += w a a' in direction order (src/spectral.cpp:105) */
    for (int d = 0; d < dirs; ++d) {
        const double* a = k->alpha + (long)d * total;
        const double* ap = k->alpha_prime + (long)d * total;
        for (long i = 0; i < total; ++i) k->loss_diag[i] += k->weight * a[i] * ap[i];
    }
    return HKO_OK;
}

void hko_kernel_free(hko_kernel* k) {
    free(k->alpha);
    free(k->alpha_prime);
    free(k->loss_diag);
    memset(k, 0, sizeof(*k));
}

/* ===================================================================== */
/* spectral collision (src/spectral.cpp:114-154, src/fft.cpp:19-81)      */
/* ===================================================================== */

static void make_phase(int n, double* ph) { /* src/fft.cpp:19-28 */
    const double w0 = -M_PI + M_PI / n;
    for (int idx = 0; idx < n; ++idx) {
        const int k = fft_frequency(idx, n);
        ph[2 * idx] = cos(-k * w0);
        ph[2 * idx + 1] = sin(-k * w0);
    }
}

static inline void cmul(double ar, double ai, double br, double bi, double* r, double* i) {
    *r = ar * br - ai * bi;
    *i = ar * bi + ai * br;
}

static void to_spectral(int n, const double* ph, const double* f, double* coeff) {
    const long total = (long)n * n * n;
    for (long i = 0; i < total; ++i) { coeff[2 * i] = f[i]; coeff[2 * i + 1] = 0.0; }
    hko_fft_3d(n, coeff, -1);
    const double scale = 1.0 / total;
    long idx = 0;
    for (int i1 = 0; i1 < n; ++i1)
        for (int i2 = 0; i2 < n; ++i2) {
            double pr, pi;
            cmul(ph[2 * i1], ph[2 * i1 + 1], ph[2 * i2], ph[2 * i2 + 1], &pr, &pi);
            pr *= scale; pi *= scale;
            for (int i3 = 0; i3 < n; ++i3, ++idx) {
                double tr, ti;
                cmul(coeff[2 * idx], coeff[2 * idx + 1], pr, pi, &tr, &ti);
                cmul(tr, ti, ph[2 * i3], ph[2 * i3 + 1], &coeff[2 * idx], &coeff[2 * idx + 1]);
            }
        }
}

static void to_nodal(int n, const double* ph, const double* coeff, double* vals) {
    long idx = 0;
    for (int i1 = 0; i1 < n; ++i1)
        for (int i2 = 0; i2 < n; ++i2) {
            double pr, pi;
            cmul(ph[2 * i1], ph[2 * i1 + 1], ph[2 * i2], ph[2 * i2 + 1], &pr, &pi);
            pi = -pi; /* conj */
            for (int i3 = 0; i3 < n; ++i3, ++idx) {
                double tr, ti;
                cmul(coeff[2 * idx], coeff[2 * idx + 1], pr, pi, &tr, &ti);
                cmul(tr, ti, ph[2 * i3], -ph[2 * i3 + 1], &vals[2 * idx], &vals[2 * idx + 1]);
            }
        }
    hko_fft_3d(n, vals, +1);
}

int hko_spectral_collision(const hko_kernel* k, const double* f, double* out, double* residue) {
    const int n = k->n;
    const long total = (long)n * n * n;
    double* ph = (double*)malloc(sizeof(double) * 2 * n);
    make_phase(n, ph);
    double* coeff = (double*)malloc(sizeof(double) * 2 * total);
    double* tmp = (double*)malloc(sizeof(double) * 2 * total);
    double* ga = (double*)malloc(sizeof(double) * 2 * total);
    double* gb = (double*)malloc(sizeof(double) * 2 * total);
    double* gain = (double*)calloc(2 * (size_t)total, sizeof(double));
    double* loss = (double*)malloc(sizeof(double) * 2 * total);

    to_spectral(n, ph, f, coeff);
    for (long i = 0; i < total; ++i) {
        tmp[2 * i] = k->loss_diag[i] * coeff[2 * i];
        tmp[2 * i + 1] = k->loss_diag[i] * coeff[2 * i + 1];
    }
    to_nodal(n, ph, tmp, loss);
    for (int d = 0; d < k->a1 * k->a2; ++d) {
        const double* a = k->alpha + (long)d * total;
        const double* ap = k->alpha_prime + (long)d * total;
        for (long i = 0; i < total; ++i) {
            tmp[2 * i] = a[i] * coeff[2 * i];
            tmp[2 * i + 1] = a[i] * coeff[2 * i + 1];
        }
        to_nodal(n, ph, tmp, ga);
        for (long i = 0; i < total; ++i) {
            tmp[2 * i] = ap[i] * coeff[2 * i];
            tmp[2 * i + 1] = ap[i] * coeff[2 * i + 1];
        }
        to_nodal(n, ph, tmp, gb);
        for (long i = 0; i < total; ++i) {
            double pr, pi;
            cmul(ga[2 * i], ga[2 * i + 1], gb[2 * i], gb[2 * i + 1], &pr, &pi);
            gain[2 * i] += pr;
            gain[2 * i + 1] += pi;
        }
    }
    double max_re = 0.0, max_im = 0.0;
    for (long i = 0; i < total; ++i) {
        const double qr = k->jacobian * (k->weight * gain[2 * i] - f[i] * loss[2 * i]);
        const double qi = k->jacobian * (k->weight * gain[2 * i + 1] - f[i] * loss[2 * i + 1]);
        out[i] = qr;
        if (fabs(qr) > max_re) max_re = fabs(qr);
        if (fabs(qi) > max_im) max_im = fabs(qi);
    }
    free(ph); free(coeff); free(tmp); free(ga); free(gb); free(gain); free(loss);
    const double denom = max_re > 1e-300 ? max_re : 1e-300;
    if (residue) *residue = max_im / denom;
    return max_im > 1e-10 * denom ? HKO_NUMERICAL_CONSISTENCY : HKO_OK;
}

/* WorkerPool-style batch (inc/threading.hpp:25-56). */
typedef struct {
    const hko_kernel* k;
    const double* f;
    double* q;
    int* st;
    double* res;
    long b, e;
} coll_job;

static void* coll_worker(void* arg) {
    coll_job* j = (coll_job*)arg;
    const long nb = (long)j->k->n * j->k->n * j->k->n;
    for (long c = j->b; c < j->e; ++c) {
        double r = 0.0;
        int s = hko_spectral_collision(j->k, j->f + c * nb, j->q + c * nb, &r);
        if (j->st) j->st[c] = s;
        if (j->res) j->res[c] = r;
    }
    return NULL;
}

int hko_collision_batch(const hko_kernel* k, const double* f, double* q, long ncells,
                        int nthreads, int* st, double* res) {
    if (ncells <= 0) return HKO_OK;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > ncells) nthreads = (int)ncells;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    coll_job jobs[256];
    const long chunk = (ncells + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].k = k; jobs[t].f = f; jobs[t].q = q; jobs[t].st = st; jobs[t].res = res;
        jobs[t].b = t * chunk;
        jobs[t].e = (t + 1) * chunk < ncells ? (t + 1) * chunk : ncells;
        if (jobs[t].b > jobs[t].e) jobs[t].b = jobs[t].e;
        if (t > 0) pthread_create(&th[t], NULL, coll_worker, &jobs[t]);
    }
    coll_worker(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    return HKO_OK;
}

/* ===================================================================== */
/* moments (src/moments.cpp)                                             */
/* ===================================================================== */

int hko_moments_of(int n, double vmax, const double* f, hko_moments* m) { /* :21-53 */
    double s0 = 0.0, sx = 0.0, sy = 0.0, sz = 0.0, s2 = 0.0;
    long idx = 0;
    for (int k1 = 0; k1 < n; ++k1) {
        const double vx = hko_node(n, vmax, k1);
        for (int k2 = 0; k2 < n; ++k2) {
            const double vy = hko_node(n, vmax, k2);
            double c0 = 0.0, cz = 0.0, c2 = 0.0;
            for (int k3 = 0; k3 < n; ++k3, ++idx) {
                const double vz = hko_node(n, vmax, k3);
                const double w = f[idx];
                c0 += w;
                cz += vz * w;
                c2 += vz * vz * w;
            }
            s0 += c0;
            sx += vx * c0;
            sy += vy * c0;
            sz += cz;
            s2 += (vx * vx + vy * vy) * c0 + c2;
        }
    }
    m->rho = s0 * hko_dvk(n, vmax);
    if (!(m->rho > 0.0)) return HKO_DEGENERATE;
    m->u[0] = sx / s0;
    m->u[1] = sy / s0;
    m->u[2] = sz / s0;
    const double usq = m->u[0] * m->u[0] + m->u[1] * m->u[1] + m->u[2] * m->u[2];
    m->T = (s2 / s0 - usq) / 3.0;
    if (!(m->T > 0.0)) return HKO_DEGENERATE;
    return HKO_OK;
}

static double energy_of(const hko_moments* m) { /* inc/moments.hpp:22 */
    const double usq = m->u[0] * m->u[0] + m->u[1] * m->u[1] + m->u[2] * m->u[2];
    return 0.5 * m->rho * usq + 1.5 * m->rho * m->T;
}

void hko_second_moment(int n, double vmax, const double* f, double s[9]) { /* :55-81 */
    double xx = 0, xy = 0, xz = 0, yy = 0, yz = 0, zz = 0;
    long idx = 0;
    for (int k1 = 0; k1 < n; ++k1) {
        const double vx = hko_node(n, vmax, k1);
        for (int k2 = 0; k2 < n; ++k2) {
            const double vy = hko_node(n, vmax, k2);
            double c0 = 0.0, cz = 0.0, c2 = 0.0;
            for (int k3 = 0; k3 < n; ++k3, ++idx) {
                const double vz = hko_node(n, vmax, k3);
                c0 += f[idx];
                cz += vz * f[idx];
                c2 += vz * vz * f[idx];
            }
            xx += vx * vx * c0;
            xy += vx * vy * c0;
            yy += vy * vy * c0;
            xz += vx * cz;
            yz += vy * cz;
            zz += c2;
        }
    }
    const double dvk = hko_dvk(n, vmax);
    s[0] = xx * dvk; s[1] = xy * dvk; s[2] = xz * dvk;
    s[3] = xy * dvk; s[4] = yy * dvk; s[5] = yz * dvk;
    s[6] = xz * dvk; s[7] = yz * dvk; s[8] = zz * dvk;
}

void hko_stress_tensor(int n, double vmax, const double* f, const hko_moments* m,
                       double theta[9]) { /* :83-86 */
    double s[9];
    hko_second_moment(n, vmax, f, s);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) theta[3 * i + j] = s[3 * i + j] / m->rho - m->u[i] * m->u[j];
}

int hko_maxwellian(const hko_moments* m, int n, double vmax, double* out) { /* :88-112 */
    if (!(m->rho > 0.0) || !(m->T > 0.0)) return HKO_DEGENERATE;
    const double inv2T = 0.5 / m->T;
    const double pref = m->rho / pow(2.0 * M_PI * m->T, 1.5);
    double ex[256], ey[256], ez[256];
    for (int k = 0; k < n; ++k) {
        const double v = hko_node(n, vmax, k);
        ex[k] = exp(-(v - m->u[0]) * (v - m->u[0]) * inv2T);
        ey[k] = exp(-(v - m->u[1]) * (v - m->u[1]) * inv2T);
        ez[k] = exp(-(v - m->u[2]) * (v - m->u[2]) * inv2T);
    }
    long idx = 0;
    for (int k1 = 0; k1 < n; ++k1) {
        const double px = pref * ex[k1];
        for (int k2 = 0; k2 < n; ++k2) {
            const double pxy = px * ey[k2];
            for (int k3 = 0; k3 < n; ++k3, ++idx) out[idx] = pxy * ez[k3];
        }
    }
    return HKO_OK;
}

/* Eigen::LLT<Matrix3d>::info() restated: fails iff a pivot x <= 0. */
static int llt_ok(const double a[9]) {
    double l[9] = {0};
    for (int k = 0; k < 3; ++k) {
        double x = a[3 * k + k];
        for (int j = 0; j < k; ++j) x -= l[3 * k + j] * l[3 * k + j];
        if (!(x > 0.0)) return 0;
        l[3 * k + k] = sqrt(x);
        for (int i = k + 1; i < 3; ++i) {
            double y = a[3 * i + k];
            for (int j = 0; j < k; ++j) y -= l[3 * i + j] * l[3 * k + j];
            l[3 * i + k] = y / l[3 * k + k];
        }
    }
    return 1;
}

static double det3(const double m[9]) { /* Eigen bruteforce_det3 */
    return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
           m[2] * (m[3] * m[7] - m[4] * m[6]);
}

static void inv3(const double m[9], double r[9]) {
    const double c00 = m[4] * m[8] - m[5] * m[7];
    const double c01 = m[5] * m[6] - m[3] * m[8];
    const double c02 = m[3] * m[7] - m[4] * m[6];
    const double det = m[0] * c00 + m[1] * c01 + m[2] * c02;
    const double id = 1.0 / det;
    r[0] = c00 * id;
    r[1] = (m[2] * m[7] - m[1] * m[8]) * id;
    r[2] = (m[1] * m[5] - m[2] * m[4]) * id;
    r[3] = c01 * id;
    r[4] = (m[0] * m[8] - m[2] * m[6]) * id;
    r[5] = (m[2] * m[3] - m[0] * m[5]) * id;
    r[6] = c02 * id;
    r[7] = (m[1] * m[6] - m[0] * m[7]) * id;
    r[8] = (m[0] * m[4] - m[1] * m[3]) * id;
}

int hko_anisotropic_gaussian(const hko_moments* m, const double theta[9], double beta, int n,
                             double vmax, double* out, int* fell_back) { /* :120-157 */
    if (fell_back) *fell_back = 0;
    double tc[9];
    const double iso = (1.0 - beta) * m->T;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) tc[3 * i + j] = (i == j ? iso : 0.0) + beta * theta[3 * i + j];
    if (!llt_ok(tc)) {
        if (fell_back) *fell_back = 1;
        return hko_maxwellian(m, n, vmax, out);
    }
    const double det = det3(tc);
    double inv[9];
    inv3(tc, inv);
    const double pref = m->rho / sqrt(pow(2.0 * M_PI, 3) * det);
    long idx = 0;
    for (int k1 = 0; k1 < n; ++k1) {
        const double dx = hko_node(n, vmax, k1) - m->u[0];
        for (int k2 = 0; k2 < n; ++k2) {
            const double dy = hko_node(n, vmax, k2) - m->u[1];
            const double qxy = inv[0] * dx * dx + 2.0 * inv[1] * dx * dy + inv[4] * dy * dy;
            const double lz = 2.0 * (inv[2] * dx + inv[5] * dy);
            for (int k3 = 0; k3 < n; ++k3, ++idx) {
                const double dz = hko_node(n, vmax, k3) - m->u[2];
                const double q = qxy + dz * (lz + inv[8] * dz);
                out[idx] = pref * exp(-0.5 * q);
            }
        }
    }
    return HKO_OK;
}

static void coupling_matrix(const double* w, int n, double vmax, const double uc[3],
                            double a[25]) { /* :164-189 */
    for (int i = 0; i < 25; ++i) a[i] = 0.0;
    long idx = 0;
    for (int k1 = 0; k1 < n; ++k1) {
        const double vx = hko_node(n, vmax, k1);
        for (int k2 = 0; k2 < n; ++k2) {
            const double vy = hko_node(n, vmax, k2);
            for (int k3 = 0; k3 < n; ++k3, ++idx) {
                const double vz = hko_node(n, vmax, k3);
                const double cx = vx - uc[0], cy = vy - uc[1], cz = vz - uc[2];
                const double c2 = cx * cx + cy * cy + cz * cz;
                const double v2 = vx * vx + vy * vy + vz * vz;
                const double psi[5] = {1.0, cx, cy, cz, c2};
                const double phi[5] = {1.0, vx, vy, vz, v2};
                const double g = w[idx];
                for (int r = 0; r < 5; ++r)
                    for (int c = 0; c < 5; ++c) a[5 * r + c] += phi[r] * psi[c] * g;
            }
        }
    }
    const double dvk = hko_dvk(n, vmax);
    for (int i = 0; i < 25; ++i) a[i] *= dvk;
}

static void invariant_moments(const double* g, int n, double vmax, double m[5]) { /* :192-213 */
    for (int i = 0; i < 5; ++i) m[i] = 0.0;
    long idx = 0;
    for (int k1 = 0; k1 < n; ++k1) {
        const double vx = hko_node(n, vmax, k1);
        for (int k2 = 0; k2 < n; ++k2) {
            const double vy = hko_node(n, vmax, k2);
            for (int k3 = 0; k3 < n; ++k3, ++idx) {
                const double vz = hko_node(n, vmax, k3);
                const double w = g[idx];
                m[0] += w;
                m[1] += vx * w;
                m[2] += vy * w;
                m[3] += vz * w;
                m[4] += (vx * vx + vy * vy + vz * vz) * w;
            }
        }
    }
    const double dvk = hko_dvk(n, vmax);
    for (int i = 0; i < 5; ++i) m[i] *= dvk;
}

/* Eigen::FullPivLU<Matrix<double,5,5>> restated: complete pivoting, rank with
 * threshold epsilon * 5 relative to the largest pivot (:215-221). */
int hko_solve5(const double a_in[25], const double rhs[5], double x[5]) {
    double a[25];
    int rp[5], cp[5];
    memcpy(a, a_in, sizeof(a));
    for (int i = 0; i < 5; ++i) { rp[i] = i; cp[i] = i; }
    double maxpivot = 0.0;
    int nonzero = 5;
    for (int k = 0; k < 5; ++k) {
        int bi = k, bj = k;
        double big = -1.0;
        for (int j = k; j < 5; ++j)     /* Eigen scans column-major */
            for (int i = k; i < 5; ++i) {
                const double v = fabs(a[5 * i + j]);
                if (v > big) { big = v; bi = i; bj = j; }
            }
        if (big == 0.0) { nonzero = k; break; }
        if (big > maxpivot) maxpivot = big;
        if (bi != k) {
            for (int j = 0; j < 5; ++j) { double t = a[5 * k + j]; a[5 * k + j] = a[5 * bi + j]; a[5 * bi + j] = t; }
            int t = rp[k]; rp[k] = rp[bi]; rp[bi] = t;
        }
        if (bj != k) {
            for (int i = 0; i < 5; ++i) { double t = a[5 * i + k]; a[5 * i + k] = a[5 * i + bj]; a[5 * i + bj] = t; }
            int t = cp[k]; cp[k] = cp[bj]; cp[bj] = t;
        }
        for (int i = k + 1; i < 5; ++i) {
            a[5 * i + k] /= a[5 * k + k];
            for (int j = k + 1; j < 5; ++j) a[5 * i + j] -= a[5 * i + k] * a[5 * k + j];
        }
    }
    const double thr = 2.220446049250313e-16 * 5.0 * maxpivot;
    int rank = 0;
    for (int i = 0; i < nonzero; ++i) rank += fabs(a[5 * i + i]) > thr;
    if (rank != 5) return HKO_DEGENERATE;
    double y[5];
    for (int i = 0; i < 5; ++i) y[i] = rhs[rp[i]];
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < i; ++j) y[i] -= a[5 * i + j] * y[j];
    for (int i = 4; i >= 0; --i) {
        for (int j = i + 1; j < 5; ++j) y[i] -= a[5 * i + j] * y[j];
        y[i] /= a[5 * i + i];
    }
    for (int i = 0; i < 5; ++i) x[cp[i]] = y[i];
    return HKO_OK;
}

int hko_match_moments(double* f, int n, double vmax, double rho, const double mom[3],
                      double energy) { /* :225-246 */
    const double uc[3] = {mom[0] / rho, mom[1] / rho, mom[2] / rho};
    const double rhs[5] = {rho, mom[0], mom[1], mom[2], 2.0 * energy};
    double a[25], x[5];
    coupling_matrix(f, n, vmax, uc, a);
    const int st = hko_solve5(a, rhs, x);
    if (st) return st;
    long idx = 0;
    for (int k1 = 0; k1 < n; ++k1) {
        const double vx = hko_node(n, vmax, k1);
        for (int k2 = 0; k2 < n; ++k2) {
            const double vy = hko_node(n, vmax, k2);
            for (int k3 = 0; k3 < n; ++k3, ++idx) {
                const double cx = vx - uc[0], cy = vy - uc[1];
                const double cz = hko_node(n, vmax, k3) - uc[2];
                const double c2 = cx * cx + cy * cy + cz * cz;
                f[idx] *= x[0] + x[1] * cx + x[2] * cy + x[3] * cz + x[4] * c2;
            }
        }
    }
    return HKO_OK;
}

int hko_remove_invariant_moments(double* q, const double* weight, int n, double vmax,
                                 const double uc[3]) { /* :248-267 */
    double a[25], rhs[5], x[5];
    coupling_matrix(weight, n, vmax, uc, a);
    invariant_moments(q, n, vmax, rhs);
    const int st = hko_solve5(a, rhs, x);
    if (st) return st;
    long idx = 0;
    for (int k1 = 0; k1 < n; ++k1) {
        const double vx = hko_node(n, vmax, k1);
        for (int k2 = 0; k2 < n; ++k2) {
            const double vy = hko_node(n, vmax, k2);
            for (int k3 = 0; k3 < n; ++k3, ++idx) {
                const double cx = vx - uc[0], cy = vy - uc[1];
                const double cz = hko_node(n, vmax, k3) - uc[2];
                const double c2 = cx * cx + cy * cy + cz * cz;
                q[idx] -= (x[0] + x[1] * cx + x[2] * cy + x[3] * cz + x[4] * c2) * weight[idx];
            }
        }
    }
    return HKO_OK;
}

void hko_realizability_matrix(const double* f, int n, double vmax, const hko_moments* m,
                              double a_bar[9], double b_bar[3], double* c_bar) { /* :269-312 */
    const double inv_sqrt_t = 1.0 / sqrt(m->T);
    double s00 = 0, s01 = 0, s02 = 0, s11 = 0, s12 = 0, s22 = 0;
    double bx = 0, by = 0, bz = 0, c4 = 0;
    long idx = 0;
    for (int k1 = 0; k1 < n; ++k1) {
        const double Vx = (hko_node(n, vmax, k1) - m->u[0]) * inv_sqrt_t;
        for (int k2 = 0; k2 < n; ++k2) {
            const double Vy = (hko_node(n, vmax, k2) - m->u[1]) * inv_sqrt_t;
            for (int k3 = 0; k3 < n; ++k3, ++idx) {
                const double Vz = (hko_node(n, vmax, k3) - m->u[2]) * inv_sqrt_t;
                const double w = f[idx];
                const double V2 = Vx * Vx + Vy * Vy + Vz * Vz;
                s00 += Vx * Vx * w;
                s01 += Vx * Vy * w;
                s02 += Vx * Vz * w;
                s11 += Vy * Vy * w;
                s12 += Vy * Vz * w;
                s22 += Vz * Vz * w;
                const double bw = 0.5 * (V2 - 5.0) * w;
                bx += bw * Vx;
                by += bw * Vy;
                bz += bw * Vz;
                const double e = 0.5 * V2 - 2.5;
                c4 += e * e * w;
            }
        }
    }
    const double scale = hko_dvk(n, vmax) / m->rho;
    double s2[9] = {s00, s01, s02, s01, s11, s12, s02, s12, s22};
    for (int i = 0; i < 9; ++i) s2[i] *= scale;
    const double tr3 = (s2[0] + s2[4] + s2[8]) / 3.0;
    for (int i = 0; i < 9; ++i) a_bar[i] = s2[i] - ((i % 4 == 0) ? tr3 : 0.0);
    b_bar[0] = bx * scale;
    b_bar[1] = by * scale;
    b_bar[2] = bz * scale;
    *c_bar = 0.4 * c4 * scale;
}

void hko_realizability_5x5(const double a_bar[9], const double b_bar[3], double c_bar,
                           double m[25]) { /* :9-19 */
    const double s = sqrt(2.0 / 5.0);
    for (int i = 0; i < 25; ++i) m[i] = 0.0;
    m[0] = 1.0;
    m[4] = m[20] = -s;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m[5 * (i + 1) + (j + 1)] = (i == j ? 1.0 : 0.0) + a_bar[3 * i + j];
    for (int i = 0; i < 3; ++i) {
        m[5 * (i + 1) + 4] = s * b_bar[i];
        m[5 * 4 + (i + 1)] = s * b_bar[i];
    }
    m[24] = c_bar;
}

/* ===================================================================== */
/* Boltzmann layer (src/boltzmann.cpp)                                   */
/* ===================================================================== */

int hko_penalized_residual(const hko_kernel* k, const double* f, double pen_coeff, double* out,
                           double* residue) { /* :9-27, spectral_collision caught-and-continued */
    const int n = k->n;
    const long nb = (long)n * n * n;
    const int cst = hko_spectral_collision(k, f, out, residue);
    hko_moments m;
    int st = hko_moments_of(n, k->vmax, f, &m);
    if (st) return st;
    const double beta = pen_coeff * m.rho;
    double* eq = (double*)malloc(sizeof(double) * nb);
    hko_maxwellian(&m, n, k->vmax, eq);
    const double mom[3] = {m.rho * m.u[0], m.rho * m.u[1], m.rho * m.u[2]};
    st = hko_match_moments(eq, n, k->vmax, m.rho, mom, energy_of(&m));
    if (!st) {
        for (long i = 0; i < nb; ++i) out[i] += beta * (f[i] - eq[i]);
        st = hko_remove_invariant_moments(out, eq, n, k->vmax, m.u);
    }
    free(eq);
    return st ? st : cst;
}

int hko_penalized_stage_solve(const double* f_star, double a, double eps, double pen_coeff,
                              int n, double vmax, double* out, hko_moments* m_out) { /* :29-45 */
    const long nb = (long)n * n * n;
    hko_moments m;
    int st = hko_moments_of(n, vmax, f_star, &m);
    if (m_out) *m_out = m;
    if (st) return st;
    const double ab = a * (pen_coeff * m.rho);
    if (ab <= 0.0) {
        memcpy(out, f_star, sizeof(double) * nb);
        return HKO_OK;
    }
    hko_maxwellian(&m, n, vmax, out);
    const double mom[3] = {m.rho * m.u[0], m.rho * m.u[1], m.rho * m.u[2]};
    st = hko_match_moments(out, n, vmax, m.rho, mom, energy_of(&m));
    if (st) return st;
    const double wf = eps / (eps + ab), wm = ab / (eps + ab);
    for (long i = 0; i < nb; ++i) out[i] = wf * f_star[i] + wm * out[i];
    return HKO_OK;
}

static long wrapi(long k, long n) { return (k % n + n) % n; }

/* PR(2,2,2) tableau (inc/imex.hpp:23-34). */
typedef struct { double a_ex10, a_im00, a_im10, a_im11, w_ex0, w_ex1, w_im0, w_im1; } pr222;
static pr222 tableau_pr222(void) {
    const double C = 1.0 / sqrt(2.0);
    const double delta = 1.0 - 1.0 / (2.0 * C);
    pr222 t = {1.0, 1.0 - C, C - delta, delta, 0.5, 0.5, 0.5, 0.5};
    return t;
}

int hko_penalized_imex_step(double* f, int nx, int ny, const hko_kernel* k, double dx,
                            double dy, double dt, const double* eps_cell, double pen_coeff,
                            double eps_weno, int nthreads) { /* src/boltzmann.cpp:47-110 */
    (void)nthreads;
    const int n = k->n;
    const double vmax = k->vmax;
    const long cells = (long)nx * ny, nb = (long)n * n * n;
    const pr222 t = tableau_pr222();
    double* stage = (double*)malloc(sizeof(double) * cells * nb);
    double* q1 = (double*)malloc(sizeof(double) * cells * nb);
    double* k1 = (double*)malloc(sizeof(double) * cells * nb);
    double* f_acc = (double*)malloc(sizeof(double) * nb);
    double* res = (double*)malloc(sizeof(double) * nb);
    double* q2 = (double*)malloc(sizeof(double) * nb);
    int first = HKO_OK;
#define NOTE(s) do { int s_ = (s); if (s_ && s_ != HKO_NUMERICAL_CONSISTENCY && !first) first = s_; } while (0)
    for (long c = 0; c < cells; ++c) {
        double* y = stage + c * nb;
        NOTE(hko_penalized_stage_solve(f + c * nb, t.a_im00 * dt, eps_cell[c], pen_coeff, n, vmax, y, NULL));
        const double inv_a = 1.0 / t.a_im00;
        for (long i = 0; i < nb; ++i) k1[c * nb + i] = (y[i] - f[c * nb + i]) * inv_a;
    }
    hko_transport_rhs_periodic(stage, nx, ny, n, vmax, dx, dy, eps_weno, q1);
    for (long c = 0; c < cells; ++c) {
        NOTE(hko_penalized_residual(k, stage + c * nb, pen_coeff, res, NULL));
        const double inv_eps = 1.0 / eps_cell[c];
        for (long i = 0; i < nb; ++i) q1[c * nb + i] += res[i] * inv_eps;
    }
    for (long c = 0; c < cells; ++c) {
        double* y = stage + c * nb;
        for (long i = 0; i < nb; ++i)
            f_acc[i] = f[c * nb + i] + dt * t.a_ex10 * q1[c * nb + i] + t.a_im10 * k1[c * nb + i];
        NOTE(hko_penalized_stage_solve(f_acc, t.a_im11 * dt, eps_cell[c], pen_coeff, n, vmax, y, NULL));
    }
    const double inv_a2 = 1.0 / t.a_im11;
    for (long c = 0; c < cells; ++c) {
        const long i = c % nx, j = c / nx;
        const double* fx[5];
        const double* fy[5];
        for (int p = -2; p <= 2; ++p) {
            fx[p + 2] = stage + (j * nx + wrapi(i + p, nx)) * nb;
            fy[p + 2] = stage + (wrapi(j + p, ny) * nx + i) * nb;
        }
        hko_transport_rhs_cell(fx, fy, n, vmax, dx, dy, eps_weno, q2);
        NOTE(hko_penalized_residual(k, stage + c * nb, pen_coeff, res, NULL));
        const double inv_eps = 1.0 / eps_cell[c];
        double* fc = f + c * nb;
        for (long kk = 0; kk < nb; ++kk) {
            const double q2k = q2[kk] + res[kk] * inv_eps;
            const double facc = fc[kk] + dt * t.a_ex10 * q1[c * nb + kk] + t.a_im10 * k1[c * nb + kk];
            const double k2 = (stage[c * nb + kk] - facc) * inv_a2;
            fc[kk] += dt * (t.w_ex0 * q1[c * nb + kk] + t.w_ex1 * q2k) + t.w_im0 * k1[c * nb + kk] +
                      t.w_im1 * k2;
        }
    }
#undef NOTE
    free(stage); free(q1); free(k1); free(f_acc); free(res); free(q2);
    return first;
}

/* ===================================================================== */
/* ES-BGK layer (src/esbgk.cpp)                                          */
/* ===================================================================== */

int hko_esbgk_stage_solve(const double* f_star, double a, double eps, double beta,
                          double nu_coeff, int n, double vmax, double* out, hko_moments* m_out,
                          int* fallback) { /* :9-45 */
    const long nb = (long)n * n * n;
    if (fallback) *fallback = 0;
    hko_moments m;
    int st = hko_moments_of(n, vmax, f_star, &m);
    if (m_out) *m_out = m;
    if (st) return st;
    const double nu = nu_coeff * m.rho;
    const double A = a * nu;
    if (A <= 0.0) {
        memcpy(out, f_star, sizeof(double) * nb);
        return HKO_OK;
    }
    const double omb = 1.0 - beta;
    double sstar[9], siso[9], sstage[9], theta[9];
    hko_second_moment(n, vmax, f_star, sstar);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            siso[3 * i + j] = m.rho * ((i == j ? m.T : 0.0) + m.u[i] * m.u[j]);
    const double denom = eps + omb * A;
    const double oa = omb * A;
    for (int i = 0; i < 9; ++i) sstage[i] = (eps * sstar[i] + oa * siso[i]) / denom;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) theta[3 * i + j] = sstage[3 * i + j] / m.rho - m.u[i] * m.u[j];
    int fb = 0;
    st = hko_anisotropic_gaussian(&m, theta, beta, n, vmax, out, &fb);
    if (fallback) *fallback = fb;
    if (st) return st;
    const double mom[3] = {m.rho * m.u[0], m.rho * m.u[1], m.rho * m.u[2]};
    st = hko_match_moments(out, n, vmax, m.rho, mom, energy_of(&m));
    if (st) return st;
    const double wf = eps / (eps + A), wg = A / (eps + A);
    for (long i = 0; i < nb; ++i) out[i] = wf * f_star[i] + wg * out[i];
    return HKO_OK;
}

int hko_esbgk_imex_step(double* f, int nx, int ny, int n, double vmax, double dx, double dy,
                        double dt, const double* eps_cell, double beta, double nu_coeff,
                        double eps_weno, int nthreads) { /* src/esbgk.cpp:47-99 */
    (void)nthreads;
    const long cells = (long)nx * ny, nb = (long)n * n * n;
    const pr222 t = tableau_pr222();
    double* stage = (double*)malloc(sizeof(double) * cells * nb);
    double* q1 = (double*)malloc(sizeof(double) * cells * nb);
    double* k1 = (double*)malloc(sizeof(double) * cells * nb);
    double* f_acc = (double*)malloc(sizeof(double) * nb);
    double* q2 = (double*)malloc(sizeof(double) * nb);
    int first = HKO_OK;
    for (long c = 0; c < cells; ++c) {
        double* y = stage + c * nb;
        int s = hko_esbgk_stage_solve(f + c * nb, t.a_im00 * dt, eps_cell[c], beta, nu_coeff, n, vmax, y, NULL, NULL);
        if (s && !first) first = s;
        const double inv_a = 1.0 / t.a_im00;
        for (long i = 0; i < nb; ++i) k1[c * nb + i] = (y[i] - f[c * nb + i]) * inv_a;
    }
    hko_transport_rhs_periodic(stage, nx, ny, n, vmax, dx, dy, eps_weno, q1);
    for (long c = 0; c < cells; ++c) {
        double* y = stage + c * nb;
        for (long i = 0; i < nb; ++i)
            f_acc[i] = f[c * nb + i] + dt * t.a_ex10 * q1[c * nb + i] + t.a_im10 * k1[c * nb + i];
        int s = hko_esbgk_stage_solve(f_acc, t.a_im11 * dt, eps_cell[c], beta, nu_coeff, n, vmax, y, NULL, NULL);
        if (s && !first) first = s;
    }
    const double inv_a2 = 1.0 / t.a_im11;
    for (long c = 0; c < cells; ++c) {
        const long i = c % nx, j = c / nx;
        const double* fx[5];
        const double* fy[5];
        for (int p = -2; p <= 2; ++p) {
            fx[p + 2] = stage + (j * nx + wrapi(i + p, nx)) * nb;
            fy[p + 2] = stage + (wrapi(j + p, ny) * nx + i) * nb;
        }
        hko_transport_rhs_cell(fx, fy, n, vmax, dx, dy, eps_weno, q2);
        double* fc = f + c * nb;
        for (long kk = 0; kk < nb; ++kk) {
            const double facc = fc[kk] + dt * t.a_ex10 * q1[c * nb + kk] + t.a_im10 * k1[c * nb + kk];
            const double k2 = (stage[c * nb + kk] - facc) * inv_a2;
            fc[kk] += dt * (t.w_ex0 * q1[c * nb + kk] + t.w_ex1 * q2[kk]) + t.w_im0 * k1[c * nb + kk] +
                      t.w_im1 * k2;
        }
    }
    free(stage); free(q1); free(k1); free(f_acc); free(q2);
    return first;
}

/* ===================================================================== */
/* indicators + regime (src/indicators.cpp, src/regime.cpp)             */
/* ===================================================================== */

void hko_spatial_derivatives(const double c[4], const double xm[4], const double xp[4],
                             const double ym[4], const double yp[4], double dx, double dy,
                             double d[11]) { /* :14-32 */
    d[0] = (xp[0] - xm[0]) / (2.0 * dx);
    d[1] = (yp[0] - ym[0]) / (2.0 * dy);
    d[2] = (xp[1] - xm[1]) / (2.0 * dx);
    d[3] = (yp[1] - ym[1]) / (2.0 * dy);
    d[4] = (xp[2] - xm[2]) / (2.0 * dx);
    d[5] = (yp[2] - ym[2]) / (2.0 * dy);
    d[6] = (xp[3] - xm[3]) / (2.0 * dx);
    d[7] = (yp[3] - ym[3]) / (2.0 * dy);
    const double inv_dxdy = 1.0 / (dx * dy);
    d[8] = (xm[0] + xp[0] + ym[0] + yp[0] - 4.0 * c[0]) * inv_dxdy;
    d[9] = (xm[1] + xp[1] + ym[1] + yp[1] - 4.0 * c[1]) * inv_dxdy;
    d[10] = (xm[2] + xp[2] + ym[2] + yp[2] - 4.0 * c[2]) * inv_dxdy;
}

void hko_v_eps1_eigenvalues(const double d[11], const double prim[4], double eps, double mu0,
                            double kappa0, double lam[3]) { /* :34-73 */
    const double dux_dx = d[2], dux_dy = d[3], duy_dx = d[4], duy_dy = d[5];
    const double dT_dx = d[6], dT_dy = d[7];
    const double a1 = (4.0 / 3.0) * dux_dx - (2.0 / 3.0) * duy_dy;
    const double a2 = dT_dx * dT_dx;
    const double b1 = dux_dy + duy_dx;
    const double b2 = dT_dx * dT_dy;
    const double c1 = (4.0 / 3.0) * duy_dy - (2.0 / 3.0) * dux_dx;
    const double c2 = dT_dy * dT_dy;
    const double h1 = -(2.0 / 3.0) * (dux_dx + duy_dy);
    const double rho = prim[0], T = prim[3];
    const double mu = mu0 * sqrt(T), kappa = kappa0 * sqrt(T);
    const double xi1 = eps * mu / (rho * T);
    const double xi2 = eps * eps * 2.0 * kappa * kappa / (3.0 * rho * rho * T * T * T);
    const double diag_gap = xi1 * (a1 - c1) + xi2 * (a2 - c2);
    const double dd = xi1 * b1 + xi2 * b2;
    const double root = sqrt(diag_gap * diag_gap + 4.0 * dd * dd);
    const double trace_term = -a1 * xi1 - a2 * xi2 - c1 * xi1 - c2 * xi2 + 2.0;
    lam[0] = 0.5 * (root + trace_term);
    lam[1] = 0.5 * (-root + trace_term);
    lam[2] = 1.0 - xi1 * h1;
}

double hko_lambda_b(const double d[11], const double prim[4], double eps, int signed_sum) {
    /* :75-87 */
    const double grad_t2 = d[6] * d[6] + d[7] * d[7];
    const double grad_u2 = d[2] * d[2] + d[3] * d[3] + d[4] * d[4] + d[5] * d[5];
    const double lap_u2 = !signed_sum ? d[9] * d[9] + d[10] * d[10]
                                      : (d[9] + d[10]) * (d[9] + d[10]);
    const double lap_rho_rel = d[8] / prim[0];
    const double T = prim[3];
    return eps * eps * (grad_t2 / T + grad_u2 + sqrt((lap_u2 + lap_rho_rel * lap_rho_rel) * (1.0 + T * T)));
}

int hko_l1_distance(const double* f, int n, double vmax, double* out) { /* :89-98 */
    hko_moments m;
    int st = hko_moments_of(n, vmax, f, &m);
    if (st) return st;
    const long nb = (long)n * n * n;
    double* eq = (double*)malloc(sizeof(double) * nb);
    hko_maxwellian(&m, n, vmax, eq);
    double acc = 0.0;
    for (long k = 0; k < nb; ++k) acc += fabs(f[k] - eq[k]);
    free(eq);
    *out = acc * hko_dvk(n, vmax);
    return HKO_OK;
}

static int near_one(const double* lam, double eta0) { /* src/regime.cpp:13-17 */
    return fabs(lam[0] - 1.0) <= eta0 && fabs(lam[1] - 1.0) <= eta0 && fabs(lam[2] - 1.0) <= eta0;
}

int hko_regime_update(int r, const double* lam, const double* lambda_b, const double* l1,
                      double eta0, double eta1, double delta0, int* out) { /* :25-52 */
    switch (r) {
    case 2:
        if (!lambda_b) return HKO_CONTRACT;
        *out = fabs(*lambda_b) > eta1 ? 2 : 1;
        return HKO_OK;
    case 1:
        if (!lambda_b) return HKO_CONTRACT;
        if (!lam) return HKO_CONTRACT;
        if (fabs(*lambda_b) > eta1) { *out = 2; return HKO_OK; }
        if (near_one(lam, eta0)) {
            if (!l1) return HKO_CONTRACT;
            *out = *l1 <= delta0 ? 0 : 1;
            return HKO_OK;
        }
        *out = 1;
        return HKO_OK;
    case 0:
        if (!lam) return HKO_CONTRACT;
        *out = near_one(lam, eta0) ? 0 : 1;
        return HKO_OK;
    default:
        return HKO_CONTRACT;
    }
}

/* ===================================================================== */
/* transport (src/transport.cpp:12-66, cweno3 src/euler.cpp:10-40)        */
/* ===================================================================== */

void hko_cweno3(double um, double uc, double up, double eps, double* left, double* right) {
    const double sl = uc - um, sr = up - uc;
    const double b = 0.5 * (up - um);
    const double c = up - 2.0 * uc + um;
    const double is_l = sl * sl, is_r = sr * sr;
    const double is_c = (13.0 / 3.0) * c * c + b * b;
    double al = 0.25 / ((eps + is_l) * (eps + is_l));
    double ac = 0.50 / ((eps + is_c) * (eps + is_c));
    double ar = 0.25 / ((eps + is_r) * (eps + is_r));
    const double inv = 1.0 / (al + ac + ar);
    al *= inv; ac *= inv; ar *= inv;
    const double pc_a = uc - c / 12.0;
    const double c0 = al * uc + ar * uc + ac * pc_a;
    const double c1 = al * sl + ar * sr + ac * b;
    const double c2 = ac * c;
    *left = c0 - 0.5 * c1 + 0.25 * c2;
    *right = c0 + 0.5 * c1 + 0.25 * c2;
}

static double upwind_flux_diff(double v, const double s[5], double eps) { /* :12-21 */
    double l, r_p, r_m;
    if (v > 0.0) {
        hko_cweno3(s[1], s[2], s[3], eps, &l, &r_p);
        hko_cweno3(s[0], s[1], s[2], eps, &l, &r_m);
        return v * (r_p - r_m);
    }
    double lp, lm, r;
    hko_cweno3(s[2], s[3], s[4], eps, &lp, &r);
    hko_cweno3(s[1], s[2], s[3], eps, &lm, &r);
    return v * (lp - lm);
}

void hko_transport_rhs_cell(const double* const fx[5], const double* const fy[5], int n,
                            double vmax, double dx, double dy, double eps_weno, double* out) {
    const double inv_dx = 1.0 / dx, inv_dy = 1.0 / dy;
    long idx = 0;
    for (int k1 = 0; k1 < n; ++k1) {
        const double vx = hko_node(n, vmax, k1);
        for (int k2 = 0; k2 < n; ++k2) {
            const double vy = hko_node(n, vmax, k2);
            for (int k3 = 0; k3 < n; ++k3, ++idx) {
                double sx[5], sy[5];
                for (int p = 0; p < 5; ++p) { sx[p] = fx[p][idx]; sy[p] = fy[p][idx]; }
                out[idx] = -upwind_flux_diff(vx, sx, eps_weno) * inv_dx -
                           upwind_flux_diff(vy, sy, eps_weno) * inv_dy;
            }
        }
    }
}

void hko_transport_rhs_periodic(const double* f, int nx, int ny, int n, double vmax, double dx,
                                double dy, double eps_weno, double* out) { /* :51-66 */
    const long nb = (long)n * n * n;
    for (long j = 0; j < ny; ++j)
        for (long i = 0; i < nx; ++i) {
            const double* fx[5];
            const double* fy[5];
            for (int p = -2; p <= 2; ++p) {
                fx[p + 2] = f + (j * nx + wrapi(i + p, nx)) * nb;
                fy[p + 2] = f + (wrapi(j + p, ny) * nx + i) * nb;
            }
            hko_transport_rhs_cell(fx, fy, n, vmax, dx, dy, eps_weno, out + (j * nx + i) * nb);
        }
}


/* ===================================================================== */
/* Layer-0 Euler (src/euler.cpp:54-189), statement order kept            */
/* ===================================================================== */
typedef struct { double rho, ux, uy, p; } HkoPrim;

static int hko_to_primitive(const double* u, double xi, HkoPrim* q) {  /* :66-82 */
    if (!(u[0] > 0.0)) return HKO_POSITIVITY;
    const double p = (xi - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
    if (!(p > 0.0)) return HKO_POSITIVITY;
    q->rho = u[0];
    q->p = p;
    q->ux = u[1] / u[0];
    q->uy = u[2] / u[0];
    return 0;
}

static void hko_to_conserved(const HkoPrim* p, double xi, double u[4]) {  /* :84-91 */
    u[0] = p->rho;
    u[1] = p->rho * p->ux;
    u[2] = p->rho * p->uy;
    u[3] = p->p / (xi - 1.0) + 0.5 * p->rho * (p->ux * p->ux + p->uy * p->uy);
}

static int hko_euler_flux(const double u[4], int axis, double xi, double f[4]) {  /* :95-108 */
    if (!(u[0] > 0.0)) return HKO_POSITIVITY;
    const double p = (xi - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
    if (!(p > 0.0)) return HKO_POSITIVITY;
    const double un = (axis == 0 ? u[1] : u[2]) / u[0];
    f[0] = u[0] * un;
    f[1] = u[1] * un;
    f[2] = u[2] * un;
    if (axis == 0) f[1] += p;
    else f[2] += p;
    f[3] = un * (u[3] + p);
    return 0;
}

static int hko_face_flux(const HkoPrim* q0, const HkoPrim* q1, const HkoPrim* q2, const HkoPrim* q3,
                         int axis, double xi, double eps, double out[4]) {  /* :124-141 */
    HkoPrim l, r;
    double dum;
    hko_cweno3(q0->rho, q1->rho, q2->rho, eps, &dum, &l.rho);
    hko_cweno3(q0->ux, q1->ux, q2->ux, eps, &dum, &l.ux);
    hko_cweno3(q0->uy, q1->uy, q2->uy, eps, &dum, &l.uy);
    hko_cweno3(q0->p, q1->p, q2->p, eps, &dum, &l.p);
    hko_cweno3(q1->rho, q2->rho, q3->rho, eps, &r.rho, &dum);
    hko_cweno3(q1->ux, q2->ux, q3->ux, eps, &r.ux, &dum);
    hko_cweno3(q1->uy, q2->uy, q3->uy, eps, &r.uy, &dum);
    hko_cweno3(q1->p, q2->p, q3->p, eps, &r.p, &dum);
    if (!(l.rho > 0.0) || !(l.p > 0.0) || !(r.rho > 0.0) || !(r.p > 0.0)) return HKO_POSITIVITY;
    /* max_wave_speed (:110-114) */
    const double ul = axis == 0 ? l.ux : l.uy, ur = axis == 0 ? r.ux : r.uy;
    const double cl = sqrt(xi * l.p / l.rho), cr = sqrt(xi * r.p / r.rho);
    const double a = fmax(fabs(ul) + cl, fabs(ur) + cr);
    double uL[4], uR[4], fl[4], fr[4];
    hko_to_conserved(&l, xi, uL);
    hko_to_conserved(&r, xi, uR);
    /* lax_friedrichs_flux (:116-121): 0.5 (fl + fr) - (0.5 a)(ur - ul) */
    int s = hko_euler_flux(uL, axis, xi, fl);
    if (s) return s;
    s = hko_euler_flux(uR, axis, xi, fr);
    if (s) return s;
    for (int k = 0; k < 4; ++k) out[k] = 0.5 * (fl[k] + fr[k]) - (0.5 * a) * (uR[k] - uL[k]);
    return 0;
}

int hko_euler_rhs_periodic(const double* u, int nx, int ny, double dx, double dy, double xi,
                           double eps_weno, double* out, long* bad_cell) {
    const long cells = (long)nx * ny;
    HkoPrim* q = malloc(sizeof(HkoPrim) * cells);
    int first = 0;
    if (bad_cell) *bad_cell = -1;
    for (long c = 0; c < cells; ++c) {
        const int s = hko_to_primitive(u + 4 * c, xi, q + c);
        if (s && !first) {
            first = s;
            if (bad_cell) *bad_cell = c;
        }
    }
    if (first) {
        free(q);
        return first;
    }
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const HkoPrim* px[5];
            const HkoPrim* py[5];
            for (int k = -2; k <= 2; ++k) {
                px[k + 2] = q + (long)j * nx + wrapi(i + k, nx);
                py[k + 2] = q + (long)wrapi(j + k, ny) * nx + i;
            }
            double fxp[4], fxm[4], fyp[4], fym[4];
            int s = hko_face_flux(px[1], px[2], px[3], px[4], 0, xi, eps_weno, fxp);
            if (!s) s = hko_face_flux(px[0], px[1], px[2], px[3], 0, xi, eps_weno, fxm);
            if (!s) s = hko_face_flux(py[1], py[2], py[3], py[4], 1, xi, eps_weno, fyp);
            if (!s) s = hko_face_flux(py[0], py[1], py[2], py[3], 1, xi, eps_weno, fym);
            const long c = (long)j * nx + i;
            if (s) {
                if (!first) {
                    first = s;
                    if (bad_cell) *bad_cell = c;
                }
                continue;
            }
            for (int k = 0; k < 4; ++k) out[4 * c + k] = -(fxp[k] - fxm[k]) / dx - (fyp[k] - fym[k]) / dy;
        }
    free(q);
    return first;
}

int hko_tvd_rk2_step_periodic(double* u, int nx, int ny, double dx, double dy, double dt,
                              double xi, double eps_weno, long* bad_cell) {
    const long n4 = 4L * nx * ny;
    double* l1 = malloc(sizeof(double) * n4);
    double* u1 = malloc(sizeof(double) * n4);
    int s = hko_euler_rhs_periodic(u, nx, ny, dx, dy, xi, eps_weno, l1, bad_cell);
    if (!s) {
        for (long i = 0; i < n4; ++i) u1[i] = u[i] + dt * l1[i];
        s = hko_euler_rhs_periodic(u1, nx, ny, dx, dy, xi, eps_weno, l1, bad_cell);
        if (!s)
            for (long i = 0; i < n4; ++i) u[i] = 0.5 * u[i] + 0.5 * u1[i] + (0.5 * dt) * l1[i];
    }
    free(l1);
    free(u1);
    return s;
}

int hko_moments_from_conserved(const double u[4], double heat_ratio, double mom5[5]) {
    if (!(u[0] > 0.0)) return HKO_POSITIVITY;
    const double p = (heat_ratio - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
    if (!(p > 0.0)) return HKO_POSITIVITY;
    mom5[0] = u[0];
    mom5[1] = u[1] / u[0];
    mom5[2] = u[2] / u[0];
    mom5[3] = 0.0;
    mom5[4] = p / u[0];
    return 0;
}

void hko_conserved_from_moments(const double mom5[5], double heat_ratio, double u[4]) {
    const double rho = mom5[0];
    u[0] = rho;
    u[1] = rho * mom5[1];
    u[2] = rho * mom5[2];
    const double u2 = mom5[1] * mom5[1] + mom5[2] * mom5[2] + mom5[3] * mom5[3];
    u[3] = rho * mom5[4] / (heat_ratio - 1.0) + 0.5 * rho * u2;
}


/* ===================================================================== */
/* Obstacles (src/grid.cpp:56-110, src/coupling.cpp:95-147)              */
/* ===================================================================== */
#define HKO_GHOST 4
static int hko_in_ghost(int nx, int ny, int i, int j) {
    return i < HKO_GHOST || i >= nx - HKO_GHOST || j < HKO_GHOST || j >= ny - HKO_GHOST;
}

static int hko_in_footprint(const hko_obstacle* s, int i, int j) {  /* src/grid.cpp:56-71 */
    if (s->shape == 1) return abs(i - s->center_i) <= s->half_i && abs(j - s->center_j) <= s->half_j;
    if (s->shape == 2) {
        const double di = i - s->center_i, dj = j - s->center_j;
        return di * di + dj * dj <= (double)s->radius * s->radius;
    }
    return 0;
}

int hko_classify_cells(int nx, int ny, const hko_obstacle* s, unsigned char* kind, long* bad_cell) {
    if (bad_cell) *bad_cell = -1;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) kind[(long)j * nx + i] = hko_in_ghost(nx, ny, i, j) ? 3 : 0;
    if (s->shape == 0) return 0;
    const int ring = 2;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const long c = (long)j * nx + i;
            if (hko_in_footprint(s, i, j)) {
                if (kind[c] == 3) { if (bad_cell) *bad_cell = c; return HKO_CONFIG; }
                kind[c] = 1;
                continue;
            }
            int near = 0;
            for (int dj = -ring; dj <= ring && !near; ++dj)
                for (int di = -ring; di <= ring && !near; ++di) near = hko_in_footprint(s, i + di, j + dj);
            if (near) {
                if (kind[c] == 3) { if (bad_cell) *bad_cell = c; return HKO_CONFIG; }
                kind[c] = 2;
            }
        }
    return 0;
}

int hko_apply_obstacle(int nx, int ny, int n, double vmax, hko_obstacle* s, signed char* r, unsigned char* kind,
                       double* hydro, double* f, double heat_ratio, int* covered, int* vacated) {
    *covered = 0;
    *vacated = 0;
    if (s->shape == 0) return 0;
    const int moving = s->move_di != 0 || s->move_dj != 0;
    s->center_i += s->move_di;
    s->center_j += s->move_dj;
    const long cells = (long)nx * ny, nb = (long)n * n * n;
    unsigned char* nk = malloc(cells);
    const int st = hko_classify_cells(nx, ny, s, nk, NULL);
    if (st) {
        free(nk);
        return moving ? HKO_SCENARIO_END : st;
    }
    /* obstacle_moments / obstacle_state (src/coupling.cpp:39-53) */
    hko_moments fm;
    fm.rho = s->rho;
    fm.u[0] = s->ux; fm.u[1] = s->uy; fm.u[2] = 0.0;
    fm.T = s->pressure / s->rho;
    const double mom5[5] = {fm.rho, fm.u[0], fm.u[1], fm.u[2], fm.T};
    double fixed[4];
    hko_conserved_from_moments(mom5, heat_ratio, fixed);
    int first = 0;
    for (long c = 0; c < cells; ++c) {
        const unsigned char before = kind[c], after = nk[c];
        if (after == 1) {
            if (before != 1) ++*covered;
            for (int k = 0; k < 4; ++k) hydro[4 * c + k] = fixed[k];
            r[c] = 2;
        } else if (before == 1) {
            ++*vacated;
            r[c] = 2;
            for (int k = 0; k < 4; ++k) hydro[4 * c + k] = fixed[k];
            const int s3 = hko_maxwellian(&fm, n, vmax, f + c * nb);
            if (s3) { first = s3; break; }  /* degenerate fixed state: throws after r, hydro */
        }
        if (after == 2 && r[c] != 2) {
            if (r[c] == 0) {
                double m5[5];
                const int s2 = hko_moments_from_conserved(hydro + 4 * c, heat_ratio, m5);
                if (s2) { first = s2; break; }  /* the reference throws mid-loop */
                hko_moments m;
                m.rho = m5[0]; m.u[0] = m5[1]; m.u[1] = m5[2]; m.u[2] = m5[3]; m.T = m5[4];
                hko_maxwellian(&m, n, vmax, f + c * nb);
            }
            r[c] = 2;
        }
        kind[c] = after;
    }
    free(nk);
    return first;
}

/* ===================================================================== */
/* Cross-layer stencil synthesis (src/coupling.cpp:57-93)                */
/* ===================================================================== */
static long hko_clamped(int nx, int ny, int i, int j) { /* SpatialGrid::clamp_interior, src/grid.cpp:12-16 */
    if (hko_in_ghost(nx, ny, i, j)) {
        const int ilo = HKO_GHOST, ihi = nx - HKO_GHOST - 1, jlo = HKO_GHOST, jhi = ny - HKO_GHOST - 1;
        i = i < ilo ? ilo : (i > ihi ? ihi : i);
        j = j < jlo ? jlo : (j > jhi ? jhi : j);
    }
    return (long)j * nx + i;
}

static hko_moments hko_fixed_moments(const hko_obstacle* s) { /* obstacle_moments, src/coupling.cpp:47-53 */
    hko_moments m;
    m.rho = s->rho;
    m.u[0] = s->ux; m.u[1] = s->uy; m.u[2] = 0.0;
    m.T = s->pressure / s->rho;
    return m;
}

int hko_synthesize_hydro_state(int nx, int ny, int n, double vmax, const hko_obstacle* s, const signed char* r,
                               const unsigned char* kind, const double* hydro, const double* f, double heat_ratio,
                               int i, int j, double out[4]) {
    const long c = hko_clamped(nx, ny, i, j);
    if (kind[c] == 1) { /* obstacle_state */
        const hko_moments m = hko_fixed_moments(s);
        const double m5[5] = {m.rho, m.u[0], m.u[1], m.u[2], m.T};
        hko_conserved_from_moments(m5, heat_ratio, out);
        return 0;
    }
    if (r[c] == 0) {
        for (int k = 0; k < 4; ++k) out[k] = hydro[4 * c + k];
        return 0;
    }
    hko_moments m;
    const int st = hko_moments_of(n, vmax, f + c * (long)n * n * n, &m);
    if (st) return st;
    const double m5[5] = {m.rho, m.u[0], m.u[1], m.u[2], m.T};
    hko_conserved_from_moments(m5, heat_ratio, out);
    return 0;
}

int hko_synthesize_distribution(int nx, int ny, int n, double vmax, const hko_obstacle* s, const signed char* r,
                                const unsigned char* kind, const double* hydro, const double* f, double heat_ratio,
                                int i, int j, double* out) {
    const long c = hko_clamped(nx, ny, i, j), nb = (long)n * n * n;
    if (kind[c] == 1) {
        const hko_moments m = hko_fixed_moments(s);
        return hko_maxwellian(&m, n, vmax, out);
    }
    if (r[c] == 0) {
        double m5[5];
        const int st = hko_moments_from_conserved(hydro + 4 * c, heat_ratio, m5);
        if (st) return st;
        hko_moments m;
        m.rho = m5[0]; m.u[0] = m5[1]; m.u[1] = m5[2]; m.u[2] = m5[3]; m.T = m5[4];
        return hko_maxwellian(&m, n, vmax, out);
    }
    memcpy(out, f + c * nb, sizeof(double) * nb);
    return 0;
}

/* ===================================================================== */
/* Hybrid time step (restatement: SPEC.md harness run_scenario, PAPER.md  */
/* Algorithm 1 + the stencil-synthesis paragraphs after it)               */
/* ===================================================================== */

static int hyb_kinetic_at(const signed char* r, int nx, int ny, long i, long j) {
    return r[wrapi(j, ny) * nx + wrapi(i, nx)] != 0;
}

int hko_hybrid_step(int nx, int ny, const hko_kernel* k, double dx, double dy, double dt, const double* eps,
                    signed char* r, double* hydro, double* f, const hko_hybrid_params* p, long counts[6]) {
    const int n = k->n;
    const double vmax = k->vmax, hr = p->heat_ratio;
    const long cells = (long)nx * ny, nb = (long)n * n * n;
    const pr222 t = tableau_pr222();
    double* mom = (double*)malloc(sizeof(double) * 5 * cells);
    double* W = (double*)malloc(sizeof(double) * 4 * cells);
    signed char* rn = (signed char*)malloc(cells);
    int st = HKO_OK;
    long n01 = 0, n10 = 0, nhalo = 0, nl[3] = {0, 0, 0};
    /* 1. indicator pass at t^n: the hydro view of every cell */
    for (long c = 0; c < cells && !st; ++c) {
        if (r[c] == 0) {
            st = hko_moments_from_conserved(hydro + 4 * c, hr, mom + 5 * c);
        } else {
            hko_moments m;
            st = hko_moments_of(n, vmax, f + c * nb, &m);
            mom[5 * c] = m.rho;
            mom[5 * c + 1] = m.u[0];
            mom[5 * c + 2] = m.u[1];
            mom[5 * c + 3] = m.u[2];
            mom[5 * c + 4] = m.T;
        }
    }
    for (long c = 0; c < cells && !st; ++c) {
        int out = r[c];
        if (p->update_regimes) { /* indicators on prim_from_moments (src/coupling.cpp:33-35) */
            const long i = c % nx, j = c / nx;
            double pc[4], xm[4], xp[4], ym[4], yp[4], d[11], lam[3], l1 = 0.0;
            const long nbr[5] = {c, j * nx + wrapi(i - 1, nx), j * nx + wrapi(i + 1, nx), wrapi(j - 1, ny) * nx + i,
                                 wrapi(j + 1, ny) * nx + i};
            double* q[5] = {pc, xm, xp, ym, yp};
            for (int e = 0; e < 5; ++e) {
                const double* m = mom + 5 * nbr[e];
                q[e][0] = m[0]; q[e][1] = m[1]; q[e][2] = m[2]; q[e][3] = m[4];
            }
            hko_spatial_derivatives(pc, xm, xp, ym, yp, dx, dy, d);
            hko_v_eps1_eigenvalues(d, pc, eps[c], p->mu0, p->kappa0, lam);
            const double lb = hko_lambda_b(d, pc, eps[c], p->signed_sum);
            if (r[c] == 1) st = hko_l1_distance(f + c * nb, n, vmax, &l1);
            if (!st) st = hko_regime_update(r[c], lam, &lb, r[c] == 1 ? &l1 : NULL, p->eta0, p->eta1, p->delta0, &out);
        }
        rn[c] = (signed char)out;
    }
    /* 2. convert_on_transition (src/regime.cpp:54-72); W = hydro view fed to layer 0 */
    for (long c = 0; c < cells && !st; ++c) {
        if (r[c] == 0) {
            memcpy(W + 4 * c, hydro + 4 * c, sizeof(double) * 4);
            if (rn[c] != 0) ++n01;
        } else {
            hko_conserved_from_moments(mom + 5 * c, hr, W + 4 * c);
            if (rn[c] == 0) {
                memcpy(hydro + 4 * c, W + 4 * c, sizeof(double) * 4);
                ++n10;
            }
        }
        ++nl[(int)rn[c]];
    }
    /* Maxwellians of the 0 -> 1 cells and of the layer-0 transport halo */
    for (long c = 0; c < cells && !st; ++c) {
        int mw = r[c] == 0 && rn[c] != 0;
        if (rn[c] == 0) {
            const long i = c % nx, j = c / nx;
            for (int dd = 1; dd <= 2 && !mw; ++dd)
                mw = hyb_kinetic_at(rn, nx, ny, i - dd, j) || hyb_kinetic_at(rn, nx, ny, i + dd, j) ||
                     hyb_kinetic_at(rn, nx, ny, i, j - dd) || hyb_kinetic_at(rn, nx, ny, i, j + dd);
            nhalo += mw;
        }
        if (mw) {
            double m5[5];
            st = hko_moments_from_conserved(hydro + 4 * c, hr, m5);
            if (!st) {
                const hko_moments m = {m5[0], {m5[1], m5[2], m5[3]}, m5[4]};
                st = hko_maxwellian(&m, n, vmax, f + c * nb);
            }
        }
    }
    /* 3. layer 0 */
    if (!st && nl[0]) {
        long bad = -1;
        st = hko_tvd_rk2_step_periodic(W, nx, ny, dx, dy, dt, hr, p->eps_weno, &bad);
        for (long c = 0; c < cells && !st; ++c)
            if (rn[c] == 0) memcpy(hydro + 4 * c, W + 4 * c, sizeof(double) * 4);
    }
    /* 4. kinetic cells: PR(2,2,2) (src/boltzmann.cpp:47-110, src/esbgk.cpp:47-99) */
    if (!st && nl[1] + nl[2]) {
        double* Y = (double*)malloc(sizeof(double) * cells * nb);
        double* q1 = (double*)malloc(sizeof(double) * cells * nb);
        double* k1 = (double*)malloc(sizeof(double) * cells * nb);
        double* fa = (double*)malloc(sizeof(double) * nb);
        double* res = (double*)malloc(sizeof(double) * nb);
        double* q2 = (double*)malloc(sizeof(double) * nb);
        memcpy(Y, f, sizeof(double) * cells * nb); /* halo cells keep their Maxwellian */
#define STAGE(fin, a, out) (rn[c] == 1 ? hko_esbgk_stage_solve(fin, a, eps[c], p->esbgk_beta, p->nu_coeff, n, vmax, out, NULL, NULL) \
                                       : hko_penalized_stage_solve(fin, a, eps[c], p->pen_coeff, n, vmax, out, NULL))
#define NOTE(x) do { int s_ = (x); if (s_ && s_ != HKO_NUMERICAL_CONSISTENCY && !st) st = s_; } while (0)
        const double inv_a = 1.0 / t.a_im00, inv_a2 = 1.0 / t.a_im11;
        for (long c = 0; c < cells; ++c) {
            if (!rn[c]) continue;
            NOTE(STAGE(f + c * nb, t.a_im00 * dt, Y + c * nb));
            for (long i = 0; i < nb; ++i) k1[c * nb + i] = (Y[c * nb + i] - f[c * nb + i]) * inv_a;
        }
        for (long c = 0; c < cells; ++c) { /* q1 = T(Y1) + res(Y1) / eps */
            if (!rn[c]) continue;
            const long i = c % nx, j = c / nx;
            const double* fx[5];
            const double* fy[5];
            for (int pp = -2; pp <= 2; ++pp) {
                fx[pp + 2] = Y + (j * nx + wrapi(i + pp, nx)) * nb;
                fy[pp + 2] = Y + (wrapi(j + pp, ny) * nx + i) * nb;
            }
            hko_transport_rhs_cell(fx, fy, n, vmax, dx, dy, p->eps_weno, q1 + c * nb);
            if (rn[c] == 2) {
                NOTE(hko_penalized_residual(k, Y + c * nb, p->pen_coeff, res, NULL));
                const double inv_eps = 1.0 / eps[c];
                for (long kk = 0; kk < nb; ++kk) q1[c * nb + kk] += res[kk] * inv_eps;
            }
        }
        for (long c = 0; c < cells; ++c) { /* Y2 */
            if (!rn[c]) continue;
            for (long i = 0; i < nb; ++i) fa[i] = f[c * nb + i] + dt * t.a_ex10 * q1[c * nb + i] + t.a_im10 * k1[c * nb + i];
            NOTE(STAGE(fa, t.a_im11 * dt, Y + c * nb));
        }
        double* fnew = (double*)malloc(sizeof(double) * cells * nb);
        for (long c = 0; c < cells; ++c) { /* final combination */
            if (!rn[c]) continue;
            const long i = c % nx, j = c / nx;
            const double* fx[5];
            const double* fy[5];
            for (int pp = -2; pp <= 2; ++pp) {
                fx[pp + 2] = Y + (j * nx + wrapi(i + pp, nx)) * nb;
                fy[pp + 2] = Y + (wrapi(j + pp, ny) * nx + i) * nb;
            }
            hko_transport_rhs_cell(fx, fy, n, vmax, dx, dy, p->eps_weno, q2);
            if (rn[c] == 2) NOTE(hko_penalized_residual(k, Y + c * nb, p->pen_coeff, res, NULL));
            const double inv_eps = 1.0 / eps[c];
            const double* fc = f + c * nb;
            for (long kk = 0; kk < nb; ++kk) {
                const double q2k = rn[c] == 2 ? q2[kk] + res[kk] * inv_eps : q2[kk];
                const double facc = fc[kk] + dt * t.a_ex10 * q1[c * nb + kk] + t.a_im10 * k1[c * nb + kk];
                const double k2 = (Y[c * nb + kk] - facc) * inv_a2;
                fnew[c * nb + kk] = fc[kk] + (dt * (t.w_ex0 * q1[c * nb + kk] + t.w_ex1 * q2k) +
                                              t.w_im0 * k1[c * nb + kk] + t.w_im1 * k2);
            }
        }
        for (long c = 0; c < cells; ++c)
            if (rn[c]) memcpy(f + c * nb, fnew + c * nb, sizeof(double) * nb);
#undef STAGE
#undef NOTE
        free(fnew); free(Y); free(q1); free(k1); free(fa); free(res); free(q2);
    }
    if (!st) memcpy(r, rn, cells);
    if (counts) {
        counts[0] = nl[0]; counts[1] = nl[1]; counts[2] = nl[2];
        counts[3] = n01; counts[4] = n10; counts[5] = nhalo;
    }
    free(mom); free(W); free(rn);
    return st;
}
