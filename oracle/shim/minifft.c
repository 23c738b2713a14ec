/* oracle/shim/minifft.c — TEST INFRASTRUCTURE (CPU oracle only).
 *
 * Recursive decimation-in-time mixed-radix Cooley-Tukey FFT (radix 4, 2 and a
 * generic odd-prime butterfly) with long-double-accurate twiddle tables, plus
 * the standard half-length packing for even-length real transforms.  Written
 * for this repository as the arithmetic behind the FFTW3 shim; it is a CPU
 * checker, never the product path.
 */
#define _GNU_SOURCE
#include "minifft.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define MF_MAXFAC 64

/* Scratch without a heap allocation per call for lengths up to 8192. */
#define MF_STACK 8192
#define SCRATCH(name, count)                                                   \
  mf_cpx name##_stack[(count) <= MF_STACK ? (count) : 1];                      \
  mf_cpx* name = (count) <= MF_STACK ? name##_stack                            \
                                     : (mf_cpx*)malloc(sizeof(mf_cpx) * (count))
#define SCRATCH_FREE(name) \
  do { if (name != name##_stack) free(name); } while (0)

struct mf_plan {
  int n;
  int sign;
  int nfac;
  int fac[2 * MF_MAXFAC]; /* (p, m) pairs */
  mf_cpx* tw;             /* tw[k] = exp(sign 2 pi i k / n) */
  int maxp;
};

struct mf_rplan {
  int n;
  mf_plan* half_f; /* n/2 forward (even n) */
  mf_plan* half_b; /* n/2 backward (even n) */
  mf_plan* full_f; /* n forward (odd n) */
  mf_plan* full_b; /* n backward (odd n) */
  mf_cpx* rtw;     /* exp(-2 pi i k / n), k < n/2 */
};

static inline mf_cpx cmul(mf_cpx a, mf_cpx b) {
  mf_cpx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}
static inline mf_cpx cadd(mf_cpx a, mf_cpx b) {
  mf_cpx r = {a.re + b.re, a.im + b.im};
  return r;
}
static inline mf_cpx csub(mf_cpx a, mf_cpx b) {
  mf_cpx r = {a.re - b.re, a.im - b.im};
  return r;
}

static mf_cpx twiddle(long k, long n, int sign) {
  /* exp(sign 2 pi i k/n) in long double, rounded once. */
  const long double pi = 3.141592653589793238462643383279502884L;
  long kk = k % n;
  if (kk < 0) kk += n;
  const long double a = 2.0L * pi * (long double)kk / (long double)n;
  mf_cpx r = {(double)cosl(a), (double)(sign * sinl(a))};
  /* exact values at the quarter points */
  if (4 * kk == n) { r.re = 0.0; r.im = (double)sign; }
  if (2 * kk == n) { r.re = -1.0; r.im = 0.0; }
  if (4 * kk == 3 * n) { r.re = 0.0; r.im = (double)-sign; }
  if (kk == 0) { r.re = 1.0; r.im = 0.0; }
  return r;
}

static void factorize(mf_plan* p) {
  int n = p->n, nf = 0;
  int m = n;
  while (m > 1) {
    int f;
    if (m % 4 == 0) f = 4;
    else if (m % 2 == 0) f = 2;
    else {
      f = 3;
      while (m % f) {
        f += 2;
        if ((long)f * f > m) { f = m; break; }
      }
    }
    m /= f;
    p->fac[2 * nf] = f;
    p->fac[2 * nf + 1] = m;
    if (f > p->maxp) p->maxp = f;
    ++nf;
  }
  p->nfac = nf;
}

mf_plan* mf_plan_create(int n, int sign) {
  if (n < 1) return NULL;
  mf_plan* p = (mf_plan*)calloc(1, sizeof(mf_plan));
  p->n = n;
  p->sign = sign < 0 ? -1 : 1;
  p->maxp = 1;
  p->tw = (mf_cpx*)malloc(sizeof(mf_cpx) * (size_t)n);
  for (int k = 0; k < n; ++k) p->tw[k] = twiddle(k, n, p->sign);
  factorize(p);
  return p;
}

void mf_plan_destroy(mf_plan* p) {
  if (!p) return;
  free(p->tw);
  free(p);
}

int mf_plan_n(const mf_plan* p) { return p->n; }

static void bfly2(mf_cpx* out, size_t fs, const mf_plan* st, int m) {
  for (int k = 0; k < m; ++k) {
    const mf_cpx t = cmul(out[m + k], st->tw[(size_t)k * fs]);
    out[m + k] = csub(out[k], t);
    out[k] = cadd(out[k], t);
  }
}

static void bfly4(mf_cpx* out, size_t fs, const mf_plan* st, int m) {
  const int fwd = st->sign < 0;
  for (int k = 0; k < m; ++k) {
    const mf_cpx a = out[k];
    const mf_cpx b = cmul(out[k + m], st->tw[(size_t)k * fs]);
    const mf_cpx c = cmul(out[k + 2 * m], st->tw[(size_t)2 * k * fs]);
    const mf_cpx d = cmul(out[k + 3 * m], st->tw[(size_t)3 * k * fs]);
    const mf_cpx ac_p = cadd(a, c), ac_m = csub(a, c);
    const mf_cpx bd_p = cadd(b, d), bd_m = csub(b, d);
    out[k] = cadd(ac_p, bd_p);
    out[k + 2 * m] = csub(ac_p, bd_p);
    if (fwd) { /* X1 = ac_m - i bd_m ; X3 = ac_m + i bd_m */
      out[k + m].re = ac_m.re + bd_m.im;
      out[k + m].im = ac_m.im - bd_m.re;
      out[k + 3 * m].re = ac_m.re - bd_m.im;
      out[k + 3 * m].im = ac_m.im + bd_m.re;
    } else {
      out[k + m].re = ac_m.re - bd_m.im;
      out[k + m].im = ac_m.im + bd_m.re;
      out[k + 3 * m].re = ac_m.re + bd_m.im;
      out[k + 3 * m].im = ac_m.im - bd_m.re;
    }
  }
}

static void bfly_generic(mf_cpx* out, size_t fs, const mf_plan* st, int m, int p) {
  mf_cpx scratch[256];
  mf_cpx* s = p <= 256 ? scratch : (mf_cpx*)malloc(sizeof(mf_cpx) * (size_t)p);
  const size_t n = (size_t)st->n;
  for (int u = 0; u < m; ++u) {
    for (int q1 = 0, k = u; q1 < p; ++q1, k += m) s[q1] = out[k];
    for (int q1 = 0, k = u; q1 < p; ++q1, k += m) {
      size_t twidx = 0;
      mf_cpx acc = s[0];
      for (int q = 1; q < p; ++q) {
        twidx += fs * (size_t)k;
        twidx %= n;
        acc = cadd(acc, cmul(s[q], st->tw[twidx]));
      }
      out[k] = acc;
    }
  }
  if (s != scratch) free(s);
}

static void work(mf_cpx* out, const mf_cpx* in, size_t fs, ptrdiff_t is, const int* fac,
                 const mf_plan* st) {
  const int p = fac[0], m = fac[1];
  if (m == 1) {
    for (int j = 0; j < p; ++j) out[j] = in[(ptrdiff_t)j * (ptrdiff_t)fs * is];
  } else {
    for (int j = 0; j < p; ++j)
      work(out + (size_t)j * m, in + (ptrdiff_t)j * (ptrdiff_t)fs * is, fs * p, is, fac + 2, st);
  }
  switch (p) {
    case 2: bfly2(out, fs, st, m); break;
    case 4: bfly4(out, fs, st, m); break;
    default: bfly_generic(out, fs, st, m, p); break;
  }
}

void mf_exec(const mf_plan* p, const mf_cpx* in, ptrdiff_t is, mf_cpx* out, ptrdiff_t os) {
  if (p->n == 1) {
    out[0] = in[0];
    return;
  }
  if (os == 1) {
    work(out, in, 1, is, p->fac, p);
    return;
  }
  SCRATCH(tmp, (size_t)p->n);
  work(tmp, in, 1, is, p->fac, p);
  for (int k = 0; k < p->n; ++k) out[(ptrdiff_t)k * os] = tmp[k];
  SCRATCH_FREE(tmp);
}

/* ---------------------------------------------------------------- real */

mf_rplan* mf_rplan_create(int n) {
  if (n < 1) return NULL;
  mf_rplan* p = (mf_rplan*)calloc(1, sizeof(mf_rplan));
  p->n = n;
  if (n % 2 == 0) {
    const int h = n / 2;
    p->half_f = mf_plan_create(h, -1);
    p->half_b = mf_plan_create(h, +1);
    p->rtw = (mf_cpx*)malloc(sizeof(mf_cpx) * (size_t)h);
    for (int k = 0; k < h; ++k) p->rtw[k] = twiddle(k, n, -1);
  } else {
    p->full_f = mf_plan_create(n, -1);
    p->full_b = mf_plan_create(n, +1);
  }
  return p;
}

void mf_rplan_destroy(mf_rplan* p) {
  if (!p) return;
  mf_plan_destroy(p->half_f);
  mf_plan_destroy(p->half_b);
  mf_plan_destroy(p->full_f);
  mf_plan_destroy(p->full_b);
  free(p->rtw);
  free(p);
}

void mf_r2c(const mf_rplan* p, const double* in, ptrdiff_t is, mf_cpx* out, ptrdiff_t os) {
  const int n = p->n;
  if (n % 2) {
    SCRATCH(a, 2 * (size_t)n);
    mf_cpx* b = a + n;
    for (int j = 0; j < n; ++j) { a[j].re = in[(ptrdiff_t)j * is]; a[j].im = 0.0; }
    mf_exec(p->full_f, a, 1, b, 1);
    for (int k = 0; k <= n / 2; ++k) out[(ptrdiff_t)k * os] = b[k];
    SCRATCH_FREE(a);
    return;
  }
  const int h = n / 2;
  SCRATCH(a, 2 * (size_t)h);
  mf_cpx* z = a + h;
  for (int j = 0; j < h; ++j) {
    a[j].re = in[(ptrdiff_t)(2 * j) * is];
    a[j].im = in[(ptrdiff_t)(2 * j + 1) * is];
  }
  mf_exec(p->half_f, a, 1, z, 1);
  /* X[k] = Xe[k] + W^k Xo[k]; Xe = (Z[k] + conj Z[h-k])/2, Xo = (Z[k] - conj Z[h-k])/(2i) */
  {
    mf_cpx x0 = {z[0].re + z[0].im, 0.0};
    mf_cpx xh = {z[0].re - z[0].im, 0.0};
    out[0] = x0;
    out[(ptrdiff_t)h * os] = xh;
  }
  for (int k = 1; k < h; ++k) {
    const mf_cpx zk = z[k], zc = {z[h - k].re, -z[h - k].im};
    const mf_cpx e = {0.5 * (zk.re + zc.re), 0.5 * (zk.im + zc.im)};
    const mf_cpx d = {0.5 * (zk.re - zc.re), 0.5 * (zk.im - zc.im)};
    const mf_cpx o = {d.im, -d.re}; /* d / i */
    out[(ptrdiff_t)k * os] = cadd(e, cmul(p->rtw[k], o));
  }
  SCRATCH_FREE(a);
}

void mf_c2r(const mf_rplan* p, const mf_cpx* in, ptrdiff_t is, double* out, ptrdiff_t os) {
  const int n = p->n;
  if (n % 2) {
    SCRATCH(a, 2 * (size_t)n);
    mf_cpx* b = a + n;
    a[0].re = in[0].re;
    a[0].im = 0.0;
    for (int k = 1; k <= n / 2; ++k) {
      a[k] = in[(ptrdiff_t)k * is];
      a[n - k].re = a[k].re;
      a[n - k].im = -a[k].im;
    }
    mf_exec(p->full_b, a, 1, b, 1);
    for (int j = 0; j < n; ++j) out[(ptrdiff_t)j * os] = b[j].re;
    SCRATCH_FREE(a);
    return;
  }
  const int h = n / 2;
  SCRATCH(a, 2 * (size_t)h);
  mf_cpx* z = a + h;
  for (int k = 0; k < h; ++k) {
    mf_cpx xk = in[(ptrdiff_t)k * is];
    mf_cpx xr = in[(ptrdiff_t)(h - k) * is];
    if (k == 0) { xk.im = 0.0; xr.im = 0.0; }
    const mf_cpx xc = {xr.re, -xr.im};
    const mf_cpx e = cadd(xk, xc);                 /* 2 Xe */
    const mf_cpx winv = {p->rtw[k].re, -p->rtw[k].im};
    const mf_cpx o = cmul(csub(xk, xc), winv);     /* 2 Xo */
    a[k].re = e.re - o.im;                         /* e + i o */
    a[k].im = e.im + o.re;
  }
  mf_exec(p->half_b, a, 1, z, 1);
  for (int j = 0; j < h; ++j) {
    out[(ptrdiff_t)(2 * j) * os] = z[j].re;
    out[(ptrdiff_t)(2 * j + 1) * os] = z[j].im;
  }
  SCRATCH_FREE(a);
}

/* ------------------------------------------------------------- threads */

static int g_threads = 0;

int mf_threads(void) {
  if (g_threads > 0) return g_threads;
  const char* e = getenv("FDEOPT_SHIM_THREADS");
  int t = e ? atoi(e) : 1;
  return t > 0 ? t : 1;
}

void mf_set_threads(int t) { g_threads = t; }

typedef struct {
  size_t lo, hi;
  void (*fn)(size_t, size_t, void*);
  void* ctx;
} mf_task;

static void* mf_thread_main(void* arg) {
  mf_task* t = (mf_task*)arg;
  t->fn(t->lo, t->hi, t->ctx);
  return NULL;
}

void mf_parallel_for(size_t count, void (*fn)(size_t, size_t, void*), void* ctx) {
  int nt = mf_threads();
  if ((size_t)nt > count) nt = (int)count;
  if (nt <= 1) {
    if (count) fn(0, count, ctx);
    return;
  }
  pthread_t th[256];
  mf_task tasks[256];
  if (nt > 256) nt = 256;
  for (int i = 0; i < nt; ++i) {
    tasks[i].lo = count * (size_t)i / (size_t)nt;
    tasks[i].hi = count * (size_t)(i + 1) / (size_t)nt;
    tasks[i].fn = fn;
    tasks[i].ctx = ctx;
  }
  for (int i = 1; i < nt; ++i) pthread_create(&th[i], NULL, mf_thread_main, &tasks[i]);
  mf_thread_main(&tasks[0]);
  for (int i = 1; i < nt; ++i) pthread_join(th[i], NULL);
}
