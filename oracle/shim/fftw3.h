/* TEST INFRASTRUCTURE ONLY -- not product code.
 *
 * Minimal stand-in for the subset of the FFTW3 API (unpinned; pkg-config `fftw3`
 * in /root/reference/proj/core/CMakeLists.txt:4) that the reference TU
 * src/fft.cpp uses, so it compiles VERBATIM from /root/reference into
 * oracle/_ref/ (FFTW is not installed in this image). Semantics restated from
 * FFTW's published definition: unnormalized DFT
 *     Y[k] = sum_j X[j] exp(sign * 2*pi*i * j*k / n),   FFTW_FORWARD = -1,
 * multi-dimensional = separable product over dims, "guru" strides in units of
 * complex elements, in-place allowed. Implementation: oracle/shim/fftw_shim.cpp.
 */
#pragma once
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

typedef struct {
  ptrdiff_t n, is, os;
} fftw_iodim64;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
fftw_plan fftw_plan_many_dft(int rank, const int* n, int howmany, fftw_complex* in,
                             const int* inembed, int istride, int idist, fftw_complex* out,
                             const int* onembed, int ostride, int odist, int sign,
                             unsigned flags);
fftw_plan fftw_plan_guru64_dft(int rank, const fftw_iodim64* dims, int howmany_rank,
                               const fftw_iodim64* howmany_dims, fftw_complex* in,
                               fftw_complex* out, int sign, unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);
int fftw_init_threads(void);
void fftw_plan_with_nthreads(int nthreads);

#ifdef __cplusplus
}
#endif
