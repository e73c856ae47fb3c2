/*
 * oracle/shims/fftw3.h -- TEST INFRASTRUCTURE ONLY (oracle checker, never shipped).
 *
 * A from-scratch implementation of the tiny subset of the FFTW3 C API that the
 * reference's FFT wrapper uses (/root/reference/proj/src/fft.cpp:20-41,66-115):
 * fftw_complex, fftw_plan, FFTW_ESTIMATE, fftw_alloc_real/complex, fftw_free,
 * fftw_plan_dft_r2c_3d, fftw_plan_dft_c2r_3d, fftw_execute, fftw_destroy_plan.
 *
 * FFTW3 is the reference's third-party arithmetic dependency; it is absent from
 * /root/reference and from this image, and its version is unpinned
 * (proj/src/CMakeLists.txt:2-3, find_library(fftw3)). This shim restates the
 * published semantics FFTW documents for these calls:
 *   - r2c_3d(n0,n1,n2): unnormalized forward DFT, exponent sign -1, output the
 *     non-redundant half spectrum, row-major (n0, n1, n2/2+1) complex.
 *   - c2r_3d(n0,n1,n2): unnormalized inverse DFT (sign +1) of a Hermitian half
 *     spectrum (the imaginary parts of self-conjugate bins are ignored).
 * Accuracy: radix-2 (power-of-two lengths) or direct DFT (other lengths) with
 * twiddles computed in long double; relative error O(1e-16 log n).
 */
#ifndef VELOREG_ORACLE_FFTW3_SHIM_H
#define VELOREG_ORACLE_FFTW3_SHIM_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

double* fftw_alloc_real(size_t n);
fftw_complex* fftw_alloc_complex(size_t n);
void fftw_free(void* p);

fftw_plan fftw_plan_dft_r2c_3d(int n0, int n1, int n2, double* in, fftw_complex* out,
                               unsigned flags);
fftw_plan fftw_plan_dft_c2r_3d(int n0, int n1, int n2, fftw_complex* in, double* out,
                               unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
