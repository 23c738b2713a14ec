/* oracle/shim/fftw3.h — TEST INFRASTRUCTURE, not product code.
 *
 * A minimal FFTW3-API shim so that the UNCHANGED reference sources
 * (/root/reference/proj/src/fft.cpp) compile and run in this container, which
 * has no FFTW3.  It declares exactly the nine FFTW symbols the reference calls
 * (fft.cpp:31-34, 41-42, 64, 68, 75-76, 83-84, 104, 108, 118-124) with FFTW's
 * published semantics:
 *   - forward sign -1, backward sign +1, every transform unnormalized;
 *   - r2c writes len/2+1 bins per row; c2r reads len/2+1 bins, ignores the
 *     imaginary part of the DC/Nyquist bins and may clobber its input;
 *   - the new-array execute functions reuse a plan's geometry on other buffers.
 * The arithmetic lives in minifft.c (mixed-radix Cooley-Tukey, any length).
 * FFTW3 itself (unpinned: proj/CMakeLists.txt:15-16) is absent here.
 */
#ifndef FDEOPT_ORACLE_FFTW3_SHIM_H
#define FDEOPT_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_DESTROY_INPUT (1U << 0)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_many_dft_r2c(int rank, const int* n, int howmany, double* in,
                                 const int* inembed, int istride, int idist, fftw_complex* out,
                                 const int* onembed, int ostride, int odist, unsigned flags);
fftw_plan fftw_plan_many_dft_c2r(int rank, const int* n, int howmany, fftw_complex* in,
                                 const int* inembed, int istride, int idist, double* out,
                                 const int* onembed, int ostride, int odist, unsigned flags);
fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out);
void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
