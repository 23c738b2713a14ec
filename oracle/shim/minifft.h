/* oracle/shim/minifft.h — TEST INFRASTRUCTURE (CPU oracle only).
 *
 * Small mixed-radix FFT used by the FFTW3 shim (fftw3.h) and by the C
 * restatement in oracle/fdeopt_oracle.c.  Unnormalized transforms with FFTW's
 * sign convention: X_k = sum_j x_j exp(sign * 2 pi i j k / n).
 */
#ifndef FDEOPT_ORACLE_MINIFFT_H
#define FDEOPT_ORACLE_MINIFFT_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double re, im;
} mf_cpx;

typedef struct mf_plan mf_plan;

/* Complex plan of any length n >= 1. */
mf_plan* mf_plan_create(int n, int sign);
void mf_plan_destroy(mf_plan* p);
int mf_plan_n(const mf_plan* p);

/* Out-of-place strided complex transform: out[k*os] = sum_j in[j*is] w^{jk}.
 * `in` and `out` must not alias.  Thread-safe for distinct buffers. */
void mf_exec(const mf_plan* p, const mf_cpx* in, ptrdiff_t is, mf_cpx* out, ptrdiff_t os);

/* Real transforms of length n (any n >= 1).
 * r2c: in has n reals (stride is), out gets n/2+1 bins (stride os).
 * c2r: in has n/2+1 bins, out gets n reals, unnormalized (x n); the imaginary
 *      parts of bin 0 and (n even) bin n/2 are ignored, as in FFTW. */
typedef struct mf_rplan mf_rplan;
mf_rplan* mf_rplan_create(int n);
void mf_rplan_destroy(mf_rplan* p);
void mf_r2c(const mf_rplan* p, const double* in, ptrdiff_t is, mf_cpx* out, ptrdiff_t os);
void mf_c2r(const mf_rplan* p, const mf_cpx* in, ptrdiff_t is, double* out, ptrdiff_t os);

/* Worker threads used by batched shim executions (env FDEOPT_SHIM_THREADS,
 * default 1).  mf_set_threads overrides the environment. */
int mf_threads(void);
void mf_set_threads(int t);

/* Run fn(lo, hi, ctx) over [0, count) split across mf_threads() threads. */
void mf_parallel_for(size_t count, void (*fn)(size_t lo, size_t hi, void* ctx), void* ctx);

#ifdef __cplusplus
}
#endif

#endif
