/* FFTW3 API subset — TEST INFRASTRUCTURE ONLY (oracle/_ref build).
 * FFTW3 is absent from this image.  These nine symbols route the
 * reference's src/fft.cpp through the oracle's radix-2 C2C transform
 * (oracle/hk_oracle.c:hko_fft_3d / hko_fft_2d), unnormalised like FFTW. */
#ifndef HK_FFTW3_SHIM_H
#define HK_FFTW3_SHIM_H
#ifdef __cplusplus
extern "C" {
#endif
typedef double fftw_complex[2];
typedef struct hk_fftw_plan_s* fftw_plan;
#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)
fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);
#ifdef __cplusplus
}
#endif
#endif
