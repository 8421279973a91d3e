/*
 * TEST INFRASTRUCTURE ONLY — not part of the product path.
 *
 * Minimal FFTW3-API shim so the UNMODIFIED reference FFT seam
 * (/root/reference/proj/src/fft.cpp:7-61) compiles without libfftw3, which is
 * absent from this image (SURVEY.md §0 finding 3, §8c).  Only the symbols the
 * reference calls are provided: fftw_plan_dft_1d (fft.cpp:26-29),
 * fftw_execute_dft (fft.cpp:50-51,57-58), the FFTW_FORWARD/BACKWARD sign
 * convention (forward = e^{-j}, unscaled; backward = e^{+j}, unscaled) and the
 * planner flags FFTW_ESTIMATE / FFTW_UNALIGNED.  The FFTW library itself is an
 * unpinned third-party dependency of the reference (proj/CMakeLists.txt:13-14);
 * this shim restates its published DFT definition, nothing more.
 */
#ifndef FCW_FFTW_SHIM_H
#define FCW_FFTW_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fcw_shim_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
