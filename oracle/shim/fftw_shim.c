/* FFTW3 API shim — TEST INFRASTRUCTURE ONLY (see fftw3.h). */
#include <stdlib.h>
#include <string.h>
#include "fftw3.h"
#include "../hk_oracle.h"

struct hk_fftw_plan_s { int rank, n, sign; fftw_complex *in, *out; };

static fftw_plan make(int rank, int n, fftw_complex* in, fftw_complex* out, int sign) {
    fftw_plan p = (fftw_plan)malloc(sizeof(*p));
    p->rank = rank; p->n = n; p->sign = sign; p->in = in; p->out = out;
    return p;
}
fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
    (void)n1; (void)n2; (void)flags; /* cubes only, as used by src/fft.cpp:35 */
    return make(3, n0, in, out, sign);
}
fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
    (void)n1; (void)flags;
    return make(2, n0, in, out, sign);
}
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    long total = p->rank == 3 ? (long)p->n * p->n * p->n : (long)p->n * p->n;
    if (in != out) memmove(out, in, sizeof(fftw_complex) * total);
    if (p->rank == 3) hko_fft_3d(p->n, (double*)out, p->sign);
    else hko_fft_2d(p->n, (double*)out, p->sign);
}
void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }
void fftw_destroy_plan(fftw_plan p) { free(p); }
