/* oracle/fdeopt_oracle.c — TEST INFRASTRUCTURE (CPU checker; never the product).
 * See fdeopt_oracle.h.  Restates /root/reference/proj/src/{problem,toeplitz,
 * circulant,admm}.cpp for (n_t, n_x1, n_x2) shapes with the minifft FFT.
 */
#define _GNU_SOURCE
#include "fdeopt_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "minifft.h"

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* or_last_error(void) { return g_err; }

/* ------------------------------------------------------------ problem */

/* problem.cpp:35-45 */
int or_frac_coeffs(double order, int count, double* g) {
  const int valid = (order > 0.0 && order < 1.0) || (order > 1.0 && order < 2.0);
  if (!valid) return fail(-1, "fractional order must lie in (0,1) or (1,2)");
  if (count < 1) return fail(-1, "coefficient count must be >= 1");
  g[0] = 1.0;
  for (int k = 1; k < count; ++k) g[k] = (1.0 - (order + 1.0) / k) * g[k - 1];
  return 0;
}

/* toeplitz.cpp:23-42 */
int or_build_riesz(double beta, int n, double h, double* col) {
  if (!(beta > 1.0 && beta < 2.0)) return fail(-1, "build_riesz: beta must lie in (1, 2)");
  if (n < 1 || !(h > 0.0)) return fail(-1, "build_riesz: bad grid parameters");
  const double c = cos(beta * M_PI / 2.0);
  if (fabs(c) < 1e-6) return fail(-1, "build_riesz: beta too close to 1");
  double* g = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  or_frac_coeffs(beta, n + 1, g);
  const double scale = -1.0 / (2.0 * c * pow(h, beta));
  col[0] = scale * 2.0 * g[1];
  if (n > 1) col[1] = scale * (g[2] + g[0]);
  for (int k = 2; k < n; ++k) col[k] = scale * g[k + 1];
  free(g);
  return 0;
}

/* toeplitz.cpp:10-21 */
int or_build_caputo(double alpha, int n, double h, double* col, double* row) {
  if (!(alpha > 0.0 && alpha < 1.0)) return fail(-1, "build_caputo: alpha must lie in (0, 1)");
  if (n < 1 || !(h > 0.0)) return fail(-1, "build_caputo: bad grid parameters");
  const double scale = 1.0 / pow(h, alpha);
  or_frac_coeffs(alpha, n, col);
  for (int k = 0; k < n; ++k) col[k] *= scale;
  for (int k = 0; k < n; ++k) row[k] = 0.0;
  row[0] = col[0];
  return 0;
}

/* toeplitz.cpp:46-58: first column of the 2n circulant, r2c half spectrum */
static void embed(int n, const double* col, const double* row, int transpose, mf_cpx* sym) {
  const double* c0 = transpose ? row : col;
  const double* r0 = transpose ? col : row;
  double* c = (double*)calloc(2 * (size_t)n, sizeof(double));
  for (int k = 0; k < n; ++k) c[k] = c0[k];
  for (int k = 1; k < n; ++k) c[n + k] = r0[n - k];
  mf_rplan* p = mf_rplan_create(2 * n);
  mf_r2c(p, c, 1, sym, 1);
  mf_rplan_destroy(p);
  free(c);
}

int or_embed_symbol(int n, const double* col, const double* row, int transpose, double* sym) {
  if (n < 1) return fail(-1, "embed_symbol: n < 1");
  embed(n, col, row, transpose, (mf_cpx*)sym);
  return 0;
}

/* circulant.cpp:10-26 with fft.cpp:111-130 (forward DFT, sign -1) */
static void tchan_eigs(int n, const double* col, const double* row, double* first_col,
                       mf_cpx* eigs) {
  double* c = first_col ? first_col : (double*)malloc(sizeof(double) * (size_t)n);
  c[0] = col[0];
  for (int i = 1; i < n; ++i) c[i] = ((n - i) * col[i] + i * row[n - i]) / n;
  mf_cpx* in = (mf_cpx*)malloc(sizeof(mf_cpx) * (size_t)n);
  for (int i = 0; i < n; ++i) { in[i].re = c[i]; in[i].im = 0.0; }
  mf_plan* p = mf_plan_create(n, -1);
  mf_exec(p, in, 1, eigs, 1);
  mf_plan_destroy(p);
  free(in);
  if (!first_col) free(c);
}

int or_tchan(int n, const double* col, const double* row, double* first_col, double* eigs) {
  if (n < 1) return fail(-1, "tchan: empty spec");
  tchan_eigs(n, col, row, first_col, (mf_cpx*)eigs);
  return 0;
}

/* ----------------------------------------------------------- operator */

struct or_op {
  int nt, n1, n2;
  double psi;
  double *tcol, *trow, *c1, *r1, *c2, *r2;
  mf_cpx *sym_t, *sym_ta, *sym_1, *sym_2;
  mf_rplan* rp[3];
};

static double* dup(const double* p, int n) {
  double* q = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(q, p, sizeof(double) * (size_t)n);
  return q;
}

static mf_cpx* mk_sym(int n, const double* col, const double* row, int tr) {
  mf_cpx* s = (mf_cpx*)malloc(sizeof(mf_cpx) * (size_t)(n + 1));
  embed(n, col, row, tr, s);
  return s;
}

or_op* or_op_create(int nt, int n1, int n2, const double* tcol, const double* trow,
                    const double* c1, const double* r1, const double* c2, const double* r2,
                    double psi) {
  if (nt < 1 || n1 < 1 || n2 < 1) {
    fail(-1, "or_op_create: bad shape");
    return NULL;
  }
  or_op* op = (or_op*)calloc(1, sizeof(or_op));
  op->nt = nt; op->n1 = n1; op->n2 = n2; op->psi = psi;
  op->tcol = dup(tcol, nt); op->trow = dup(trow, nt);
  op->c1 = dup(c1, n1); op->r1 = dup(r1, n1);
  op->c2 = dup(c2, n2); op->r2 = dup(r2, n2);
  op->sym_t = mk_sym(nt, tcol, trow, 0);
  op->sym_ta = mk_sym(nt, tcol, trow, 1);
  op->sym_1 = mk_sym(n1, c1, r1, 0);
  op->sym_2 = mk_sym(n2, c2, r2, 0);
  op->rp[0] = mf_rplan_create(2 * nt);
  op->rp[1] = mf_rplan_create(2 * n1);
  op->rp[2] = mf_rplan_create(2 * n2);
  return op;
}

void or_op_destroy(or_op* op) {
  if (!op) return;
  free(op->tcol); free(op->trow); free(op->c1); free(op->r1); free(op->c2); free(op->r2);
  free(op->sym_t); free(op->sym_ta); free(op->sym_1); free(op->sym_2);
  for (int m = 0; m < 3; ++m) mf_rplan_destroy(op->rp[m]);
  free(op);
}

/* Fibre-parallel loops: the fibres / lines of one mode are independent and
 * each writes its own output elements, so splitting them over threads gives
 * results bit-identical to the serial loop (the reductions stay serial). */
static int g_or_threads = 1;
void or_set_threads(int t) { g_or_threads = t < 1 ? 1 : t; }
int or_get_threads(void) { return g_or_threads; }

typedef void (*or_range_fn)(void* ctx, size_t lo, size_t hi);
typedef struct { or_range_fn fn; void* ctx; size_t lo, hi; } or_task;
static void* or_task_main(void* p) {
  or_task* t = (or_task*)p;
  t->fn(t->ctx, t->lo, t->hi);
  return NULL;
}
static void par_for(size_t n, or_range_fn fn, void* ctx) {
  int nt = g_or_threads;
  if ((size_t)nt > n) nt = (int)n;
  if (nt <= 1) { fn(ctx, 0, n); return; }
  or_task* tasks = (or_task*)malloc(sizeof(or_task) * (size_t)nt);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nt);
  for (int i = 0; i < nt; ++i) {
    tasks[i].fn = fn; tasks[i].ctx = ctx;
    tasks[i].lo = n * (size_t)i / (size_t)nt; tasks[i].hi = n * (size_t)(i + 1) / (size_t)nt;
  }
  for (int i = 1; i < nt; ++i) pthread_create(&th[i], NULL, or_task_main, &tasks[i]);
  or_task_main(&tasks[0]);
  for (int i = 1; i < nt; ++i) pthread_join(th[i], NULL);
  free(tasks); free(th);
}

/* toeplitz.cpp:124-172 for one mode: fibre f of mode m starts at base(f) with
 * stride; pack into a 2n row, r2c, x symbol, c2r, out += scale/(2n) * row. */
typedef struct {
  const or_op* op; int mode; const double* x; double* out; const mf_cpx* sym; double scale;
} mode_ctx;

static void apply_mode_range(void* vctx, size_t f0, size_t f1) {
  const mode_ctx* c = (const mode_ctx*)vctx;
  const or_op* op = c->op;
  const int mode = c->mode;
  const size_t n1 = (size_t)op->n1, n2 = (size_t)op->n2;
  const int n = mode == 0 ? op->nt : (mode == 1 ? op->n1 : op->n2);
  const int len = 2 * n, sl = n + 1;
  const size_t stride = mode == 0 ? n1 * n2 : (mode == 1 ? n2 : 1);
  double* row = (double*)malloc(sizeof(double) * (size_t)len);
  mf_cpx* spec = (mf_cpx*)malloc(sizeof(mf_cpx) * (size_t)sl);
  const double w = c->scale / len;
  for (size_t f = f0; f < f1; ++f) {
    size_t base;
    if (mode == 0) base = f;                                  /* f = i*n2 + j */
    else if (mode == 1) base = (f / n2) * n1 * n2 + f % n2;   /* f = k*n2 + j */
    else base = f * n2;                                       /* f = k*n1 + i */
    for (int t = 0; t < len; ++t) row[t] = 0.0;
    for (int t = 0; t < n; ++t) row[t] = c->x[base + (size_t)t * stride];
    mf_r2c(op->rp[mode], row, 1, spec, 1);
    for (int b = 0; b < sl; ++b) {
      const mf_cpx a = spec[b], s = c->sym[b];
      spec[b].re = a.re * s.re - a.im * s.im;
      spec[b].im = a.re * s.im + a.im * s.re;
    }
    mf_c2r(op->rp[mode], spec, 1, row, 1);
    for (int t = 0; t < n; ++t) c->out[base + (size_t)t * stride] += w * row[t];
  }
  free(row);
  free(spec);
}

static void apply_mode(const or_op* op, int mode, const double* x, double* out,
                       const mf_cpx* sym, double scale) {
  const int n = mode == 0 ? op->nt : (mode == 1 ? op->n1 : op->n2);
  const size_t nfib = (size_t)op->nt * op->n1 * op->n2 / (size_t)n;
  mode_ctx c = {op, mode, x, out, sym, scale};
  par_for(nfib, apply_mode_range, &c);
}

/* toeplitz.cpp:174-182 */
int or_op_apply(const or_op* op, const double* x, double* out, int adjoint) {
  const size_t N = (size_t)op->nt * op->n1 * op->n2;
  for (size_t i = 0; i < N; ++i) out[i] = 0.0;
  apply_mode(op, 0, x, out, adjoint ? op->sym_ta : op->sym_t, op->psi);
  apply_mode(op, 1, x, out, op->sym_1, -op->psi);
  apply_mode(op, 2, x, out, op->sym_2, -op->psi);
  return 0;
}

/* Independent check: T[i][j] = t_{i-j}; col for i >= j, row for j > i
 * (toeplitz.hpp:14-19); transpose swaps col/row. */
static void direct_mode(const or_op* op, int mode, const double* x, double* out,
                        const double* col, const double* row, double scale) {
  const size_t n1 = (size_t)op->n1, n2 = (size_t)op->n2, nt = (size_t)op->nt;
  const int n = mode == 0 ? op->nt : (mode == 1 ? op->n1 : op->n2);
  const size_t nfib = nt * n1 * n2 / (size_t)n;
  const size_t stride = mode == 0 ? n1 * n2 : (mode == 1 ? n2 : 1);
  for (size_t f = 0; f < nfib; ++f) {
    size_t base;
    if (mode == 0) base = f;
    else if (mode == 1) base = (f / n2) * n1 * n2 + f % n2;
    else base = f * n2;
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int j = 0; j < n; ++j) {
        const double t = i >= j ? col[i - j] : row[j - i];
        acc += t * x[base + (size_t)j * stride];
      }
      out[base + (size_t)i * stride] += scale * acc;
    }
  }
}

int or_op_apply_direct(const or_op* op, const double* x, double* out, int adjoint) {
  const size_t N = (size_t)op->nt * op->n1 * op->n2;
  for (size_t i = 0; i < N; ++i) out[i] = 0.0;
  if (adjoint) direct_mode(op, 0, x, out, op->trow, op->tcol, op->psi);
  else direct_mode(op, 0, x, out, op->tcol, op->trow, op->psi);
  direct_mode(op, 1, x, out, op->c1, op->r1, -op->psi);
  direct_mode(op, 2, x, out, op->c2, op->r2, -op->psi);
  return 0;
}

/* ----------------------------------------------------- preconditioner */

struct or_pc {
  int nt, n1, n2;
  double rho, delta, gamma, psi;
  mf_cpx *lt, *l1, *l2;
  double* lam_s;
  mf_plan *f[3], *b[3];
};

/* circulant.cpp:76-90 then the ctor 28-41 */
or_pc* or_pc_assemble(const or_op* op, double rho, double delta, double gamma) {
  if (!(rho > 0.0) || !(delta > 0.0) || !(gamma > 0.0)) {
    fail(-1, "CirculantPreconditioner: scalars must be positive");
    return NULL;
  }
  or_pc* pc = (or_pc*)calloc(1, sizeof(or_pc));
  pc->nt = op->nt; pc->n1 = op->n1; pc->n2 = op->n2;
  pc->rho = rho; pc->delta = delta; pc->gamma = gamma; pc->psi = op->psi;
  pc->lt = (mf_cpx*)malloc(sizeof(mf_cpx) * (size_t)op->nt);
  pc->l1 = (mf_cpx*)malloc(sizeof(mf_cpx) * (size_t)op->n1);
  pc->l2 = (mf_cpx*)malloc(sizeof(mf_cpx) * (size_t)op->n2);
  tchan_eigs(op->nt, op->tcol, op->trow, NULL, pc->lt);
  tchan_eigs(op->n1, op->c1, op->r1, NULL, pc->l1);
  tchan_eigs(op->n2, op->c2, op->r2, NULL, pc->l2);
  const size_t N = (size_t)op->nt * op->n1 * op->n2;
  pc->lam_s = (double*)malloc(sizeof(double) * N);
  const double psi = op->psi;
  const double m2 = 1.0 / (rho * (gamma / (psi * psi) + 1.0 / delta)) + delta / rho;
  const double base = rho * (1.0 + 1.0 / delta);
  for (int k = 0; k < op->nt; ++k)
    for (int i = 0; i < op->n1; ++i)
      for (int j = 0; j < op->n2; ++j) {
        /* lam_b = psi * (lam_t[k] - (lam_1[i] + lam_2[j])) */
        const double sr = pc->l1[i].re + pc->l2[j].re, si = pc->l1[i].im + pc->l2[j].im;
        const double br = psi * (pc->lt[k].re - sr), bi = psi * (pc->lt[k].im - si);
        pc->lam_s[((size_t)k * op->n1 + i) * op->n2 + j] = base + (br * br + bi * bi) / m2;
      }
  const int dims[3] = {op->nt, op->n1, op->n2};
  for (int a = 0; a < 3; ++a) {
    pc->f[a] = mf_plan_create(dims[a], -1);
    pc->b[a] = mf_plan_create(dims[a], +1);
  }
  return pc;
}

void or_pc_destroy(or_pc* pc) {
  if (!pc) return;
  free(pc->lt); free(pc->l1); free(pc->l2); free(pc->lam_s);
  for (int a = 0; a < 3; ++a) { mf_plan_destroy(pc->f[a]); mf_plan_destroy(pc->b[a]); }
  free(pc);
}

typedef struct { const or_pc* pc; mf_cpx* d; int inverse, axis; } fft3_ctx;

static void fft3_range(void* vctx, size_t l0, size_t l1) {
  const fft3_ctx* c = (const fft3_ctx*)vctx;
  const or_pc* pc = c->pc;
  const size_t nt = (size_t)pc->nt, n1 = (size_t)pc->n1, n2 = (size_t)pc->n2;
  const size_t dims[3] = {nt, n1, n2};
  const int axis = c->axis;
  const mf_plan* p = c->inverse ? pc->b[axis] : pc->f[axis];
  const size_t len = dims[axis];
  mf_cpx* a = (mf_cpx*)malloc(sizeof(mf_cpx) * 2 * len);
  mf_cpx* b = a + len;
  for (size_t line = l0; line < l1; ++line) {
    size_t base, stride;
    if (axis == 2) { base = line * n2; stride = 1; }
    else if (axis == 1) { base = (line / n2) * n1 * n2 + line % n2; stride = n2; }
    else { base = line; stride = n1 * n2; }
    for (size_t t = 0; t < len; ++t) a[t] = c->d[base + t * stride];
    mf_exec(p, a, 1, b, 1);
    for (size_t t = 0; t < len; ++t) c->d[base + t * stride] = b[t];
  }
  free(a);
}

static void fft3(const or_pc* pc, mf_cpx* d, int inverse) {
  const size_t dims[3] = {(size_t)pc->nt, (size_t)pc->n1, (size_t)pc->n2};
  const size_t N = dims[0] * dims[1] * dims[2];
  for (int axis = 2; axis >= 0; --axis) {
    fft3_ctx c = {pc, d, inverse, axis};
    par_for(N / dims[axis], fft3_range, &c);
  }
}

/* circulant.cpp:49-67 */
int or_pc_solve(const or_pc* pc, const double* r, double* z) {
  const size_t N = (size_t)pc->nt * pc->n1 * pc->n2;
  mf_cpx* f = (mf_cpx*)malloc(sizeof(mf_cpx) * N);
  for (size_t i = 0; i < N; ++i) { f[i].re = r[i]; f[i].im = 0.0; }
  fft3(pc, f, 0);
  for (size_t i = 0; i < N; ++i) { f[i].re /= pc->lam_s[i]; f[i].im /= pc->lam_s[i]; }
  fft3(pc, f, 1);
  const double inv_n = 1.0 / (double)N;
  for (size_t i = 0; i < N; ++i) z[i] = f[i].re * inv_n;
  free(f);
  return 0;
}

int or_pc_lam_s(const or_pc* pc, double* out) {
  memcpy(out, pc->lam_s, sizeof(double) * (size_t)pc->nt * pc->n1 * pc->n2);
  return 0;
}

int or_pc_eigs(const or_pc* pc, double* lt, double* l1, double* l2) {
  if (lt) memcpy(lt, pc->lt, sizeof(mf_cpx) * (size_t)pc->nt);
  if (l1) memcpy(l1, pc->l1, sizeof(mf_cpx) * (size_t)pc->n1);
  if (l2) memcpy(l2, pc->l2, sizeof(mf_cpx) * (size_t)pc->n2);
  return 0;
}

/* --------------------------------------------------------------- ADMM */

struct or_admm {
  const or_op* op;
  const or_pc* pc;
  size_t N;
  double rho, delta, psi, tol_primal, inner_tol_floor, inner_tol_factor, fixed_tol;
  int max_inner, warm_start;
  double y_lo, y_hi, v_lo, v_hi;
  double *diag_j, *diag_j2, *m2, *a2_inv, *ybar;
  double *y, *v, *z_y, *z_v, *p, *w_y, *w_v, *By;
  double inner_tol;
  int iteration, converged, stagnations;
};

static double* zeros(size_t n) { return (double*)calloc(n, sizeof(double)); }

/* admm.cpp:52-79 with objective_weights problem.cpp:60-68 */
or_admm* or_admm_create(const or_op* op, const or_pc* pc, double gamma, double rho, double delta,
                        double y_lo, double y_hi, double u_lo, double u_hi, double tol_primal,
                        int max_inner, double inner_tol_floor, double inner_tol_factor,
                        double fixed_tol, int warm_start, const double* ybar) {
  or_admm* a = (or_admm*)calloc(1, sizeof(or_admm));
  a->op = op; a->pc = pc;
  a->N = (size_t)op->nt * op->n1 * op->n2;
  a->rho = rho; a->delta = delta; a->psi = op->psi; a->tol_primal = tol_primal;
  a->inner_tol_floor = inner_tol_floor; a->inner_tol_factor = inner_tol_factor;
  a->fixed_tol = fixed_tol; a->max_inner = max_inner; a->warm_start = warm_start;
  a->y_lo = y_lo; a->y_hi = y_hi; a->v_lo = a->psi * u_lo; a->v_hi = a->psi * u_hi;
  const size_t N = a->N;
  a->diag_j = zeros(N); a->diag_j2 = zeros(N); a->m2 = zeros(N); a->a2_inv = zeros(N);
  a->ybar = zeros(N);
  const size_t last = (size_t)(op->nt - 1) * op->n1 * op->n2;
  const double g_over_psi2 = gamma / (a->psi * a->psi);
  for (size_t i = 0; i < N; ++i) {
    a->diag_j[i] = i >= last ? 0.5 : 1.0;
    a->diag_j2[i] = g_over_psi2 * a->diag_j[i];
    a->a2_inv[i] = 1.0 / (rho * (a->diag_j2[i] + 1.0 / delta));
    a->m2[i] = a->a2_inv[i] + delta / rho;
  }
  if (ybar) memcpy(a->ybar, ybar, sizeof(double) * N);
  a->y = zeros(N); a->v = zeros(N); a->z_y = zeros(N); a->z_v = zeros(N);
  a->p = zeros(N); a->w_y = zeros(N); a->w_v = zeros(N); a->By = zeros(N);
  a->inner_tol = inner_tol_factor * inner_tol_floor;
  return a;
}

void or_admm_destroy(or_admm* a) {
  if (!a) return;
  double* bufs[] = {a->diag_j, a->diag_j2, a->m2, a->a2_inv, a->ybar, a->y, a->v,
                    a->z_y, a->z_v, a->p, a->w_y, a->w_v, a->By};
  for (size_t i = 0; i < sizeof bufs / sizeof bufs[0]; ++i) free(bufs[i]);
  free(a);
}

size_t or_admm_size(const or_admm* a) { return a->N; }

static double** field(const or_admm* a, int f) {
  static __thread double* tmp;
  or_admm* m = (or_admm*)a;
  switch (f) {
    case 0: return &m->y;
    case 1: return &m->v;
    case 2: return &m->z_y;
    case 3: return &m->z_v;
    case 4: return &m->p;
    case 5: return &m->w_y;
    case 6: return &m->w_v;
    case 7: return &m->ybar;
    case 8: return &m->diag_j;
    case 9: return &m->diag_j2;
    case 10: return &m->m2;
    case 11: return &m->a2_inv;
    case 12: return &m->By;
    default: tmp = NULL; return &tmp;
  }
}

int or_admm_get(const or_admm* a, int f, double* out) {
  double** p = field(a, f);
  if (!*p) return fail(-1, "or_admm_get: bad field");
  memcpy(out, *p, sizeof(double) * a->N);
  return 0;
}

int or_admm_set(or_admm* a, int f, const double* in) {
  double** p = field(a, f);
  if (!*p) return fail(-1, "or_admm_set: bad field");
  memcpy(*p, in, sizeof(double) * a->N);
  return 0;
}

static double dot(const double* a, const double* b, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* admm.cpp:87-98 */
int or_admm_apply_S(or_admm* a, const double* x, double* out) {
  const size_t N = a->N;
  double* bx = zeros(N);
  double* btm = zeros(N);
  or_op_apply(a->op, x, bx, 0);
  for (size_t i = 0; i < N; ++i) bx[i] /= a->m2[i];
  or_op_apply(a->op, bx, btm, 1);
  for (size_t i = 0; i < N; ++i) out[i] = a->rho * (a->diag_j[i] + 1.0 / a->delta) * x[i] + btm[i];
  free(bx);
  free(btm);
  return 0;
}

/* admm.cpp:100-119 (g == 0) */
int or_admm_build_rhs(or_admm* a, double* rhs, double* r_cache) {
  const size_t N = a->N;
  const double rho = a->rho, delta = a->delta;
  double* r = r_cache ? r_cache : zeros(N);
  double* tmp = zeros(N);
  for (size_t i = 0; i < N; ++i)
    r[i] = -a->psi * 0.0 + (delta / rho) * a->p[i] +
           a->a2_inv[i] * (rho * (-a->w_v[i] + a->z_v[i] / delta) + (1.0 - rho) * a->p[i]);
  for (size_t i = 0; i < N; ++i) tmp[i] = (1.0 - rho) * a->p[i] - r[i] / a->m2[i];
  or_op_apply(a->op, tmp, rhs, 1);
  for (size_t i = 0; i < N; ++i)
    rhs[i] += rho * (a->diag_j[i] * a->ybar[i] - a->w_y[i] + a->z_y[i] / delta);
  free(tmp);
  if (!r_cache) free(r);
  return 0;
}

/* admm.cpp:121-169 */
int or_admm_pcg(or_admm* a, const double* rhs, double* x, double tol, int max_inner,
                double* result) {
  const size_t N = a->N;
  const double nb = sqrt(dot(rhs, rhs, N));
  if (nb == 0.0) {
    for (size_t i = 0; i < N; ++i) x[i] = 0.0;
    result[0] = 0; result[1] = 1; result[2] = 0.0;
    return 0;
  }
  double *r = zeros(N), *z = zeros(N), *p = zeros(N), *q = zeros(N);
  int rc = 0;
  if (sqrt(dot(x, x, N)) == 0.0) {
    memcpy(r, rhs, sizeof(double) * N);
  } else {
    or_admm_apply_S(a, x, q);
    for (size_t i = 0; i < N; ++i) r[i] = rhs[i] - q[i];
  }
  or_pc_solve(a->pc, r, z);
  memcpy(p, z, sizeof(double) * N);
  double rz = dot(r, z, N);
  int it;
  for (it = 1; it <= max_inner; ++it) {
    or_admm_apply_S(a, p, q);
    const double pq = dot(p, q, N);
    if (!isfinite(pq) || pq <= 0.0) { rc = fail(-2, "pcg: operator lost positive definiteness"); goto done; }
    const double al = rz / pq;
    for (size_t i = 0; i < N; ++i) { x[i] += al * p[i]; r[i] -= al * q[i]; }
    double rn = sqrt(dot(r, r, N));
    if (!isfinite(rn)) { rc = fail(-2, "pcg: non-finite residual"); goto done; }
    if (rn <= tol * nb) {
      or_admm_apply_S(a, x, q);
      for (size_t i = 0; i < N; ++i) r[i] = rhs[i] - q[i];
      rn = sqrt(dot(r, r, N));
      if (rn <= tol * nb) {
        result[0] = it; result[1] = 1; result[2] = rn / nb;
        goto done;
      }
    }
    or_pc_solve(a->pc, r, z);
    const double rz_next = dot(r, z, N);
    const double beta = rz_next / rz;
    rz = rz_next;
    for (size_t i = 0; i < N; ++i) p[i] = z[i] + beta * p[i];
  }
  or_admm_apply_S(a, x, q);
  for (size_t i = 0; i < N; ++i) q[i] = rhs[i] - q[i];
  result[0] = max_inner; result[1] = 0; result[2] = sqrt(dot(q, q, N)) / nb;
done:
  free(r); free(z); free(p); free(q);
  return rc;
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* admm.cpp:221-233 */
int or_admm_dual_inf(or_admm* a, double* out) {
  const size_t N = a->N;
  double* btp = zeros(N);
  or_op_apply(a->op, a->p, btp, 1);
  double s1 = 0.0, s2 = 0.0;
  for (size_t i = 0; i < N; ++i) {
    s1 = fmax(s1, fabs(a->diag_j[i] * (a->y[i] - a->ybar[i]) + btp[i] + a->w_y[i]));
    s2 = fmax(s2, fabs(a->diag_j2[i] * a->v[i] + a->p[i] + a->w_v[i]));
  }
  free(btp);
  *out = fmax(s1, s2);
  return 0;
}

/* admm.cpp:245-277 */
int or_admm_step(or_admm* a, double* rec) {
  const size_t N = a->N;
  const double rho = a->rho, delta = a->delta;
  double* rhs = zeros(N);
  double* r_cache = zeros(N);
  or_admm_build_rhs(a, rhs, r_cache);
  if (!a->warm_start) memset(a->y, 0, sizeof(double) * N);
  double res[3];
  const double tol = a->fixed_tol > 0.0 ? a->fixed_tol : a->inner_tol;
  int rc = or_admm_pcg(a, rhs, a->y, tol, a->max_inner, res);
  if (rc) { free(rhs); free(r_cache); return rc; }
  a->stagnations = res[1] != 0.0 ? 0 : a->stagnations + 1;
  or_op_apply(a->op, a->y, a->By, 0);
  /* recover_vp admm.cpp:171-183 (p~ discarded), z_update 185-191, dual_update 193-200 */
  for (size_t i = 0; i < N; ++i) {
    const double pt = (a->By[i] + r_cache[i]) / a->m2[i];
    a->v[i] = a->a2_inv[i] * (-pt - rho * a->w_v[i] + (rho / delta) * a->z_v[i] + (1.0 - rho) * a->p[i]);
  }
  for (size_t i = 0; i < N; ++i) {
    a->z_y[i] = clampd(a->y[i] + delta * a->w_y[i], a->y_lo, a->y_hi);
    a->z_v[i] = clampd(a->v[i] + delta * a->w_v[i], a->v_lo, a->v_hi);
  }
  const double step = rho / delta;
  for (size_t i = 0; i < N; ++i) {
    a->p[i] += step * (a->By[i] + a->v[i] - a->psi * 0.0);
    a->w_y[i] += step * (a->y[i] - a->z_y[i]);
    a->w_v[i] += step * (a->v[i] - a->z_v[i]);
  }
  ++a->iteration;
  free(rhs);
  free(r_cache);
  for (size_t i = 0; i < N; ++i)
    if (!isfinite(a->y[i]) || !isfinite(a->v[i]) || !isfinite(a->p[i]))
      return fail(-2, "admm: non-finite iterate");
  /* check_termination admm.cpp:202-219 */
  double r_eq = 0.0, r_y = 0.0, r_v = 0.0;
  for (size_t i = 0; i < N; ++i) {
    r_eq = fmax(r_eq, fabs(a->By[i] + a->v[i] - a->psi * 0.0));
    r_y = fmax(r_y, fabs(a->y[i] - a->z_y[i]));
    r_v = fmax(r_v, fabs(a->v[i] - a->z_v[i]));
  }
  const double r_u = r_v / a->psi;
  a->converged = r_eq <= a->tol_primal && r_y <= a->tol_primal && r_u <= a->tol_primal;
  double mn = r_eq < r_y ? r_eq : r_y;
  if (r_u < mn) mn = r_u;
  a->inner_tol = a->inner_tol_factor * fmax(mn, a->inner_tol_floor);
  double dinf;
  or_admm_dual_inf(a, &dinf);
  rec[0] = a->iteration; rec[1] = r_eq; rec[2] = r_y; rec[3] = r_u; rec[4] = dinf;
  rec[5] = res[0]; rec[6] = a->inner_tol; rec[7] = a->converged;
  return 0;
}

int or_admm_objective(const or_admm* a, double* out) {
  double s1 = 0.0, s2 = 0.0;
  for (size_t i = 0; i < a->N; ++i) {
    const double d = a->y[i] - a->ybar[i];
    s1 += a->diag_j[i] * d * d;
    s2 += a->diag_j2[i] * a->v[i] * a->v[i];
  }
  *out = 0.5 * s1 + 0.5 * s2;
  return 0;
}
