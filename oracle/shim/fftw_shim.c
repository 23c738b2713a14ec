/* oracle/shim/fftw_shim.c — TEST INFRASTRUCTURE (CPU oracle only).
 *
 * Implements the nine FFTW3 entry points the reference calls (see fftw3.h)
 * on top of minifft.c.  Batched executions are split over
 * FDEOPT_SHIM_THREADS worker threads (default 1), the way FFTW's threaded
 * planner would; the reference's own loops around the FFTs stay serial.
 */
#include "fftw3.h"

#include <stdlib.h>
#include <string.h>

#include "minifft.h"

enum { K_R2C = 1, K_C2R = 2, K_C1D = 3, K_C3D = 4 };

struct fftw_plan_s {
  int kind;
  int n;       /* transform length (1-D kinds) */
  int howmany; /* batch count */
  int istride, idist, ostride, odist;
  int dims[3];
  int sign;
  void* in;
  void* out;
  mf_rplan* rp;
  mf_plan* cp[3];
};

static fftw_plan alloc_plan(int kind) {
  fftw_plan p = (fftw_plan)calloc(1, sizeof(struct fftw_plan_s));
  p->kind = kind;
  return p;
}

fftw_plan fftw_plan_many_dft_r2c(int rank, const int* n, int howmany, double* in,
                                 const int* inembed, int istride, int idist, fftw_complex* out,
                                 const int* onembed, int ostride, int odist, unsigned flags) {
  (void)inembed; (void)onembed; (void)flags;
  if (rank != 1 || n[0] < 1 || howmany < 1) return NULL;
  fftw_plan p = alloc_plan(K_R2C);
  p->n = n[0];
  p->howmany = howmany;
  p->istride = istride; p->idist = idist; p->ostride = ostride; p->odist = odist;
  p->in = in; p->out = out;
  p->rp = mf_rplan_create(n[0]);
  return p;
}

fftw_plan fftw_plan_many_dft_c2r(int rank, const int* n, int howmany, fftw_complex* in,
                                 const int* inembed, int istride, int idist, double* out,
                                 const int* onembed, int ostride, int odist, unsigned flags) {
  (void)inembed; (void)onembed; (void)flags;
  if (rank != 1 || n[0] < 1 || howmany < 1) return NULL;
  fftw_plan p = alloc_plan(K_C2R);
  p->n = n[0];
  p->howmany = howmany;
  p->istride = istride; p->idist = idist; p->ostride = ostride; p->odist = odist;
  p->in = in; p->out = out;
  p->rp = mf_rplan_create(n[0]);
  return p;
}

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
  (void)flags;
  if (n0 < 1 || n1 < 1 || n2 < 1) return NULL;
  fftw_plan p = alloc_plan(K_C3D);
  p->dims[0] = n0; p->dims[1] = n1; p->dims[2] = n2;
  p->sign = sign;
  p->in = in; p->out = out;
  for (int a = 0; a < 3; ++a) p->cp[a] = mf_plan_create(p->dims[a], sign);
  return p;
}

fftw_plan fftw_plan_dft_1d(int n, fftw_complex* in, fftw_complex* out, int sign, unsigned flags) {
  (void)flags;
  if (n < 1) return NULL;
  fftw_plan p = alloc_plan(K_C1D);
  p->n = n;
  p->sign = sign;
  p->in = in; p->out = out;
  p->cp[0] = mf_plan_create(n, sign);
  return p;
}

/* ------------------------------------------------------------ execute */

typedef struct {
  const struct fftw_plan_s* p;
  void* in;
  void* out;
} batch_ctx;

static void r2c_rows(size_t lo, size_t hi, void* vctx) {
  batch_ctx* c = (batch_ctx*)vctx;
  const struct fftw_plan_s* p = c->p;
  const double* in = (const double*)c->in;
  mf_cpx* out = (mf_cpx*)c->out;
  for (size_t r = lo; r < hi; ++r)
    mf_r2c(p->rp, in + r * (size_t)p->idist, p->istride, out + r * (size_t)p->odist, p->ostride);
}

static void c2r_rows(size_t lo, size_t hi, void* vctx) {
  batch_ctx* c = (batch_ctx*)vctx;
  const struct fftw_plan_s* p = c->p;
  const mf_cpx* in = (const mf_cpx*)c->in;
  double* out = (double*)c->out;
  for (size_t r = lo; r < hi; ++r)
    mf_c2r(p->rp, in + r * (size_t)p->idist, p->istride, out + r * (size_t)p->odist, p->ostride);
}

void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out) {
  batch_ctx c = {p, in, out};
  if ((size_t)p->howmany * (size_t)p->n < 65536)
    r2c_rows(0, (size_t)p->howmany, &c);
  else
    mf_parallel_for((size_t)p->howmany, r2c_rows, &c);
}

void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
  batch_ctx c = {p, in, out};
  if ((size_t)p->howmany * (size_t)p->n < 65536)
    c2r_rows(0, (size_t)p->howmany, &c);
  else
    mf_parallel_for((size_t)p->howmany, c2r_rows, &c);
}

/* 3-D: transform lines along each axis in turn (axis 2 contiguous). */
typedef struct {
  const struct fftw_plan_s* p;
  mf_cpx* data;
  int axis;
} axis_ctx;

static void axis_lines(size_t lo, size_t hi, void* vctx) {
  axis_ctx* c = (axis_ctx*)vctx;
  const int n0 = c->p->dims[0], n1 = c->p->dims[1], n2 = c->p->dims[2];
  const int len = c->p->dims[c->axis];
  const mf_plan* pl = c->p->cp[c->axis];
  mf_cpx* buf = (mf_cpx*)malloc(sizeof(mf_cpx) * 2 * (size_t)len);
  mf_cpx* res = buf + len;
  for (size_t line = lo; line < hi; ++line) {
    size_t base;
    ptrdiff_t stride;
    if (c->axis == 2) { base = line * (size_t)n2; stride = 1; }
    else if (c->axis == 1) {
      const size_t k = line / (size_t)n2, j = line % (size_t)n2;
      base = k * (size_t)n1 * n2 + j; stride = n2;
    } else { base = line; stride = (ptrdiff_t)n1 * n2; }
    (void)n0;
    for (int t = 0; t < len; ++t) buf[t] = c->data[base + (size_t)t * stride];
    mf_exec(pl, buf, 1, res, 1);
    for (int t = 0; t < len; ++t) c->data[base + (size_t)t * stride] = res[t];
  }
  free(buf);
}

static void exec_3d(const struct fftw_plan_s* p, mf_cpx* in, mf_cpx* out) {
  const size_t N = (size_t)p->dims[0] * p->dims[1] * p->dims[2];
  if (in != out) memcpy(out, in, sizeof(mf_cpx) * N);
  for (int axis = 2; axis >= 0; --axis) {
    axis_ctx c = {p, out, axis};
    const size_t lines = N / (size_t)p->dims[axis];
    if (N < 65536) axis_lines(0, lines, &c);
    else mf_parallel_for(lines, axis_lines, &c);
  }
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  if (p->kind == K_C3D) {
    exec_3d(p, (mf_cpx*)in, (mf_cpx*)out);
  } else if (p->kind == K_C1D) {
    if (in == out) {
      mf_cpx* tmp = (mf_cpx*)malloc(sizeof(mf_cpx) * (size_t)p->n);
      memcpy(tmp, in, sizeof(mf_cpx) * (size_t)p->n);
      mf_exec(p->cp[0], tmp, 1, (mf_cpx*)out, 1);
      free(tmp);
    } else {
      mf_exec(p->cp[0], (const mf_cpx*)in, 1, (mf_cpx*)out, 1);
    }
  }
}

void fftw_execute(const fftw_plan p) {
  switch (p->kind) {
    case K_R2C: fftw_execute_dft_r2c(p, (double*)p->in, (fftw_complex*)p->out); break;
    case K_C2R: fftw_execute_dft_c2r(p, (fftw_complex*)p->in, (double*)p->out); break;
    default: fftw_execute_dft(p, (fftw_complex*)p->in, (fftw_complex*)p->out); break;
  }
}

void fftw_destroy_plan(fftw_plan p) {
  if (!p) return;
  mf_rplan_destroy(p->rp);
  for (int a = 0; a < 3; ++a) mf_plan_destroy(p->cp[a]);
  free(p);
}
