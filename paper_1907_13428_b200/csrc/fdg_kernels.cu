// fdg_kernels.cu — sm_100a kernels of the fractional-diffusion PCG hot path.
//
// Reference hot path (/root/reference/proj/src):
//   ConstraintOperator::apply_mode / apply  toeplitz.cpp:124-182
//   CirculantPreconditioner::solve          circulant.cpp:49-67
//   apply_S / pcg vector algebra            admm.cpp:87-98, 121-169
//   build_rhs, recover_vp, z_update, dual_update, check_termination,
//   dual_infeasibility                      admm.cpp:100-119, 171-233
//
// Data layout in HBM: x[(k*n1 + i)*n2 + j], fp64, time outermost, x2
// contiguous (problem.hpp:29-39).  No packing/zero-fill buffers: zero padding
// and truncation of the circulant embedding happen in registers.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "fdg_fft.cuh"
#include "fdg_internal.h"
#include "fdg_passes.cuh"
#include "fdg_conv.cuh"
#include "fdg_launch.cuh"
#include "fdg_reduce.cuh"

namespace fdg {

// ============================================================ elementwise
namespace {
constexpr int EW_THREADS = 256;
inline unsigned ew_grid(size_t N) {
  size_t b = (N + EW_THREADS - 1) / EW_THREADS;
  const size_t cap = 148 * 8;
  return (unsigned)(b < 1 ? 1 : (b > cap ? cap : b));
}
}  // namespace

#define GRID_STRIDE(i, N) for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < (N); i += (size_t)gridDim.x * blockDim.x)

__global__ void k_copy(double* dst, const double* src, size_t N) {
  GRID_STRIDE(i, N) dst[i] = src[i];
}
__global__ void k_fill(double* dst, double v, size_t N) {
  GRID_STRIDE(i, N) dst[i] = v;
}
// 3-level preconditioner for level sizes without a radix plan (any n; the
// reference's Fft3D takes any n, circulant.cpp:49-67): the same operator
// H^-1 diag(1 / (N lambda_S)) H axis by axis with dense real Hartley
// transforms, out[o][k][c] = sum_j cas(2 pi j k / n) in[o][j][c] (cas table
// in shared memory, O(n) per element): the correctness path for small or
// irregular grids, not a bandwidth path.
__global__ void k_cas_axis(const double* in, double* out, long O, int n, long C, const double* cas) {
  extern __shared__ double tab[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) tab[i] = cas[i];
  __syncthreads();
  GRID_STRIDE(e, (size_t)O * n * C) {
    const size_t r = e / (size_t)C;
    const long c = (long)(e - r * (size_t)C);
    const int k = (int)(r % (size_t)n);
    const size_t o = r / (size_t)n;
    const double* src = in + o * (size_t)n * C + c;
    double acc = 0.0;
    int m = 0;
    for (int j = 0; j < n; ++j) {
      acc = fma(tab[m], src[(size_t)j * C], acc);
      m += k;
      if (m >= n) m -= n;
    }
    out[e] = acc;
  }
}

// h *= 1 / (N lambda_S[k, i, j]) with lambda_S from the three 1-D eigenvalue
// vectors (circulant.cpp:28-41, 62-64; the formula of k_t_filter).
__global__ void k_lams_scale(double* h, PcTables pt) {
  const size_t sl = (size_t)pt.n1 * pt.n2;
  GRID_STRIDE(e, (size_t)pt.nt * sl) {
    const int k = (int)(e / sl);
    const size_t ij = e - (size_t)k * sl;
    const int i = (int)(ij / pt.n2), j = (int)(ij - (size_t)i * pt.n2);
    const double2 lt = pt.lam_t[k], l1 = pt.lam_1[i], l2 = pt.lam_2[j];
    const double bx = pt.psi * (lt.x - (l1.x + l2.x)), by = pt.psi * (lt.y - (l1.y + l2.y));
    const double ls = pt.base + (bx * bx + by * by) * pt.inv_m2;
    h[e] *= pt.inv_total / ls;
  }
}

cudaError_t launch_cas_axis(cudaStream_t st, LaunchCounter* lc, const double* in, double* out, long O, int n,
                            long C, const double* cas) {
  count(lc);
  const size_t smem = sizeof(double) * (size_t)n;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(k_cas_axis, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_cas_axis<<<ew_grid((size_t)O * n * C), EW_THREADS, smem, st>>>(in, out, O, n, C, cas);
  return cudaGetLastError();
}

cudaError_t launch_lams_scale(cudaStream_t st, LaunchCounter* lc, double* h, const PcTables& pt) {
  count(lc);
  k_lams_scale<<<ew_grid((size_t)pt.nt * pt.n1 * pt.n2), EW_THREADS, 0, st>>>(h, pt);
  return cudaGetLastError();
}

// *flag = 1 if some x[i] is not +-0 (NaN included): norm2(x) != 0 without a
// reduction (admm.cpp:131), for the host-buffer solve's x0 check.
__global__ void k_any_nonzero(const double* x, size_t N, int* flag) {
  bool nz = false;
  GRID_STRIDE(i, N) nz |= !(x[i] == 0.0);
  if (__syncthreads_or(nz) && threadIdx.x == 0) *flag = 1;
}
__global__ void k_dot(const double* a, const double* b, size_t N, RedSlot red) {
  __shared__ double scratch[32];
  double s = 0.0;
  GRID_STRIDE(i, N) s += a[i] * (b ? b[i] : a[i]);
  double vv[1] = {s};
  block_reduce<RED_SUM, 1>(vv, scratch);
  grid_finalize<RED_SUM, 1>(vv, red, scratch);
}
// admm.cpp:148-150 and 163: x += a p; p = z + beta p
__global__ void k_cg_update(double* x, double* p, const double* z, size_t N, const double* an,
                            const double* ad, const double* bn, const double* bd, int update_x) {
  const double alpha = update_x ? (*an / *ad) : 0.0;
  const double beta = *bn / *bd;
  GRID_STRIDE(i, N) {
    const double pi = p[i];
    if (update_x) x[i] += alpha * pi;
    p[i] = z[i] + beta * pi;
  }
}
__global__ void k_axpy_dev(double* x, const double* p, size_t N, const double* an, const double* ad,
                           const int* guard) {
  pdl_trigger();
  pdl_wait();
  if (guard && *reinterpret_cast<const volatile int*>(guard)) return;
  const double alpha = *an / *ad;
  GRID_STRIDE(i, N) x[i] += alpha * p[i];
}
__global__ void k_residual(double* r, const double* b, const double* q, size_t N, RedSlot red) {
  __shared__ double scratch[32];
  double s = 0.0;
  GRID_STRIDE(i, N) {
    const double v = b[i] - q[i];
    r[i] = v;
    s += v * v;
  }
  double vv[1] = {s};
  block_reduce<RED_SUM, 1>(vv, scratch);
  grid_finalize<RED_SUM, 1>(vv, red, scratch);
}
__global__ void k_scale_by_slice(double* out, const double* x, const double* coef, size_t slice, size_t N) {
  GRID_STRIDE(i, N) out[i] = coef[i / slice] * x[i];
}

// admm.cpp:100-119 (g == 0): r = (delta/rho) p + A2^-1 (rho(-w_v + z_v/delta) + (1-rho) p);
// tmp = (1-rho) p - r / m2
__global__ void k_rhs_pre(AdmmScalars s, const double* p, const double* w_v, const double* z_v,
                          const double* a2inv, const double* m2, double* r_cache, double* tmp, size_t slice,
                          size_t N) {
  GRID_STRIDE(i, N) {
    const size_t k = i / slice;
    const double pi = p[i];
    const double r = (s.delta / s.rho) * pi + a2inv[k] * (s.rho * (-w_v[i] + z_v[i] / s.delta) + (1.0 - s.rho) * pi);
    r_cache[i] = r;
    tmp[i] = (1.0 - s.rho) * pi - r / m2[k];
  }
}
// rhs += rho (J ybar - w_y + z_y / delta)
__global__ void k_rhs_post(AdmmScalars s, double* rhs, const double* ybar, const double* w_y, const double* z_y,
                           const double* diag_j, size_t slice, size_t N) {
  GRID_STRIDE(i, N) {
    const size_t k = i / slice;
    rhs[i] += s.rho * (diag_j[k] * ybar[i] - w_y[i] + z_y[i] / s.delta);
  }
}

__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}

// recover_vp (171-183), z_update (185-191), dual_update (193-200),
// finiteness (267-269) and check_termination maxima (202-219), per element in
// the reference's order.
__global__ void k_admm_update(AdmmScalars s, const double* y, double* v, double* z_y, double* z_v, double* p,
                              double* w_y, double* w_v, const double* By, const double* r_cache,
                              const double* a2inv, const double* m2, size_t slice, size_t N, RedSlot red) {
  __shared__ double scratch[4 * 32];
  double r_eq = 0.0, r_y = 0.0, r_v = 0.0, bad = 0.0;
  const double step = s.rho / s.delta;
  GRID_STRIDE(i, N) {
    const size_t k = i / slice;
    const double by = By[i], yi = y[i], pi = p[i], wv = w_v[i], zv = z_v[i], wy = w_y[i];
    const double pt = (by + r_cache[i]) / m2[k];
    const double vi = a2inv[k] * (-pt - s.rho * wv + (s.rho / s.delta) * zv + (1.0 - s.rho) * pi);
    const double zy_n = clampd(yi + s.delta * wy, s.y_lo, s.y_hi);
    const double zv_n = clampd(vi + s.delta * wv, s.v_lo, s.v_hi);
    const double p_n = pi + step * (by + vi - s.psi * 0.0);
    const double wy_n = wy + step * (yi - zy_n);
    const double wv_n = wv + step * (vi - zv_n);
    v[i] = vi;
    z_y[i] = zy_n;
    z_v[i] = zv_n;
    p[i] = p_n;
    w_y[i] = wy_n;
    w_v[i] = wv_n;
    if (!isfinite(yi) || !isfinite(vi) || !isfinite(p_n)) bad = 1.0;
    r_eq = fmax(r_eq, fabs(by + vi - s.psi * 0.0));
    r_y = fmax(r_y, fabs(yi - zy_n));
    r_v = fmax(r_v, fabs(vi - zv_n));
  }
  double vv[4] = {r_eq, r_y, r_v, bad};
  block_reduce<RED_MAX, 4>(vv, scratch);
  grid_finalize<RED_MAX, 4>(vv, red, scratch);
}

// admm.cpp:221-233
__global__ void k_dual_inf(const double* y, const double* ybar, const double* btp, const double* w_y,
                           const double* v, const double* p, const double* w_v, const double* diag_j,
                           const double* diag_j2, size_t slice, size_t N, RedSlot red) {
  __shared__ double scratch[2 * 32];
  double s1 = 0.0, s2 = 0.0;
  GRID_STRIDE(i, N) {
    const size_t k = i / slice;
    s1 = fmax(s1, fabs(diag_j[k] * (y[i] - ybar[i]) + btp[i] + w_y[i]));
    s2 = fmax(s2, fabs(diag_j2[k] * v[i] + p[i] + w_v[i]));
  }
  double vv[2] = {s1, s2};
  block_reduce<RED_MAX, 2>(vv, scratch);
  grid_finalize<RED_MAX, 2>(vv, red, scratch);
}

__global__ void k_objective(const double* y, const double* ybar, const double* v, const double* diag_j,
                            const double* diag_j2, size_t slice, size_t N, RedSlot red) {
  __shared__ double scratch[2 * 32];
  double s1 = 0.0, s2 = 0.0;
  GRID_STRIDE(i, N) {
    const size_t k = i / slice;
    const double d = y[i] - ybar[i];
    s1 += diag_j[k] * d * d;
    s2 += diag_j2[k] * v[i] * v[i];
  }
  double vv[2] = {s1, s2};
  block_reduce<RED_SUM, 2>(vv, scratch);
  grid_finalize<RED_SUM, 2>(vv, red, scratch);
}

// ================================================================ dispatch
// Per-length launchers live in fdg_launch.cuh and are instantiated in the
// fdg_inst_*.cu translation units (parallel compilation).
template <int MODE>
static cudaError_t dispatch_row(cudaStream_t st, int L, const RowArgs& a) {
  switch (L) {
#define X(LL) \
  case LL: return run_row<LL, MODE>(st, a);
    FDG_POW2_CASES(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

template <int MODE>
static cudaError_t dispatch_col(cudaStream_t st, int L, const ColArgs& a) {
  switch (L) {
#define X(LL) \
  case LL: return run_col<LL, MODE>(st, a);
    FDG_POW2_CASES(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_row_apply(cudaStream_t st, LaunchCounter* lc, const double* x, double* out, int nt, int n1,
                             int n2, const AxisSym& s2, double scale, const TimeFactor& tf, double psi,
                             bool adjoint, const double2* chirp_in) {
  RowArgs a{};
  a.chirp_in = chirp_in;
  a.x = x;
  a.out = out;
  a.nt = nt;
  a.n1 = n1;
  a.n = n2;
  a.sym = s2.sym;
  a.sym_re = s2.sym_re;
  a.tw = s2.tw;
  a.twh = s2.twh;
  a.twist = s2.twist;
  a.tw256 = s2.tw256;
  a.twq = s2.twq;
  a.scale = scale;
  a.tkind = (tf.kind == 1 && tf.c1 != 0.0) ? 1 : 0;  // no neighbour term without a sub-diagonal
  a.tc0 = 0.0;  // folded into the x2 symbol (fdg_api.cu ax2s)
  a.tc1 = psi * tf.c1;
  a.tdir = adjoint ? +1 : -1;
  count(lc);
  return dispatch_row<0>(st, s2.L, a);
}

cudaError_t launch_row_s_out(cudaStream_t st, LaunchCounter* lc, const double* w, const double* vp, double* q_out,
                             double* r, int nt, int n1, int n2, const AxisSym& s2, double scale,
                             const TimeFactor& tf, double psi, const double* alpha_num, const double* alpha_den,
                             RedSlot red, const int* guard, const double* r_in) {
  RowArgs a{};
  a.guard = guard;
  a.r_in = r_in;
  a.x = w;
  a.vp = vp;
  a.q_out = q_out;
  a.r = r;
  a.nt = nt;
  a.n1 = n1;
  a.n = n2;
  a.sym = s2.sym;
  a.sym_re = s2.sym_re;
  a.tw = s2.tw;
  a.twh = s2.twh;
  a.twist = s2.twist;
  a.tw256 = s2.tw256;
  a.twq = s2.twq;
  a.scale = scale;
  a.tkind = (tf.kind == 1 && tf.c1 != 0.0) ? 1 : 0;  // no neighbour term without a sub-diagonal
  a.tc0 = 0.0;  // folded into the x2 symbol (fdg_api.cu ax2s)
  a.tc1 = psi * tf.c1;
  a.tdir = +1;
  a.a_num = alpha_num;
  a.a_den = alpha_den;
  a.red = red;
  count(lc);
  return dispatch_row<1>(st, s2.L, a);
}

cudaError_t launch_row_fused(cudaStream_t st, LaunchCounter* lc, const double* z, const double* dold, double* dnew,
                             double* xs, double* u, int nt, int n1, int n2, const AxisSym& s2, double scale,
                             const TimeFactor& tf, double psi, const double* a_num, const double* a_den,
                             const double* b_num, const double* b_den, bool first, bool upd_x,
                             const int* guard) {
  RowArgs a{};
  a.guard = guard;
  a.z = z;
  a.dold = dold;
  a.dnew = dnew;
  a.xs = xs;
  a.out = u;
  a.nt = nt;
  a.n1 = n1;
  a.n = n2;
  a.sym = s2.sym;
  a.sym_re = s2.sym_re;
  a.tw = s2.tw;
  a.twh = s2.twh;
  a.twist = s2.twist;
  a.tw256 = s2.tw256;
  a.twq = s2.twq;
  a.scale = scale;
  a.tkind = (tf.kind == 1 && tf.c1 != 0.0) ? 1 : 0;  // no neighbour term without a sub-diagonal
  a.tc0 = 0.0;
  a.tc1 = psi * tf.c1;
  a.tdir = -1;
  a.a_num = a_num;
  a.a_den = a_den;
  a.b_num = b_num;
  a.b_den = b_den;
  a.first = first ? 1 : 0;
  a.upd_x = upd_x ? 1 : 0;
  count(lc);
  return dispatch_row<2>(st, s2.L, a);
}

cudaError_t launch_col_acc(cudaStream_t st, LaunchCounter* lc, const double* x, const double* acc, double* out,
                           int O, int n, int C, const AxisSym& s, double scale, bool adjoint) {
  ColArgs a{};
  a.x = x;
  a.acc = acc;
  a.out = out;
  a.O = O;
  a.n = n;
  a.C = C;
  a.sym = adjoint ? s.sym_adj : s.sym;
  a.sym_re = adjoint ? s.sym_adj_re : s.sym_re;
  a.tw = s.tw;
  a.twh = s.twh;
  a.twist = s.twist;
  a.tw256 = s.tw256;
  a.twq = s.twq;
  a.scale = scale;
  count(lc);
  return dispatch_col<0>(st, s.L, a);
}

cudaError_t launch_col_s_mid(cudaStream_t st, LaunchCounter* lc, const double* p, const double* u, double* w,
                             double* vp, int nt, int n1, int n2, const AxisSym& s1, double scale,
                             const double* inv_m2, const double* a1, RedSlot red, const int* guard) {
  ColArgs a{};
  a.guard = guard;
  a.x = p;
  a.acc = u;
  a.w = w;
  a.out = vp;
  a.O = nt;
  a.n = n1;
  a.C = n2;
  a.sym = s1.sym;
  a.sym_re = s1.sym_re;
  a.tw = s1.tw;
  a.twh = s1.twh;
  a.twist = s1.twist;
  a.tw256 = s1.tw256;
  a.twq = s1.twq;
  a.scale = scale;
  a.inv_m2 = inv_m2;
  a.a1 = a1;
  a.red = red;
  count(lc);
  return dispatch_col<2>(st, s1.L, a);
}

#define FDG_POW2_CASES1(X) X(1) FDG_POW2_CASES(X)

cudaError_t launch_hartley_row(cudaStream_t st, LaunchCounter* lc, const double* in, double* out, int F, int n,
                               const double2* tw, const double* rdot, RedSlot red, const int* guard) {
  count(lc);
  switch (n) {
#define X(NN) \
  case NN: return run_hrow<NN>(st, in, out, F, tw, rdot, red, guard);
    FDG_POW2_CASES1(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_hartley_col(cudaStream_t st, LaunchCounter* lc, double* data, int O, int n, int C,
                               const double2* tw, const int* guard) {
  count(lc);
  switch (n) {
#define X(NN) \
  case NN: return run_hcol<NN>(st, data, O, C, tw, guard);
    FDG_POW2_CASES1(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_t_filter(cudaStream_t st, LaunchCounter* lc, double* data, const PcTables& pt, const int* guard) {
  count(lc);
  switch (pt.nt) {
#define X(NN) \
  case NN: return run_tf<NN>(st, data, pt, guard);
    FDG_POW2_CASES1(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

// One thread: publish (pq, |r|^2) for the host and raise the pause flag when
// the host has to intervene before the next (speculatively enqueued)
// iteration may run: breakdown checks and the reference's true-residual
// confirmation (admm.cpp:143-158).
__global__ void k_pcg_control(const double* pq, const double* rr, double tol_nb2, double* out, int* pause,
                              const int* guard, double seq) {
  pdl_trigger();
  pdl_wait();
  if (guard && *reinterpret_cast<const volatile int*>(guard)) return;
  const double p = *pq, r2 = *rr;
  // slightly looser than the host's |r| <= tol |b| so that every host-side
  // candidate has paused the stream; the host re-checks with the reference's
  // exact comparison
  const bool bad = !isfinite(p) || p <= 0.0 || !isfinite(r2);
  const bool stop = bad || r2 <= tol_nb2 * (1.0 + 1e-12);
  if (stop) *pause = 1;
  // out is host-mapped pinned memory: the values, then (after a system
  // fence) the sequence number the host spins on
  volatile double* o = out;
  o[0] = p;
  o[1] = r2;
  o[2] = stop ? 1.0 : 0.0;
  __threadfence_system();
  o[3] = seq;
}

cudaError_t launch_pcg_control(cudaStream_t st, LaunchCounter* lc, const double* pq, const double* rr,
                               double tol_nb2, double* out, int* pause, const int* guard, double seq) {
  count(lc);
#if FDG_CARVEOUT
  static int dev_set = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev_set != dev) {
    cudaFuncSetAttribute(k_pcg_control, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
    dev_set = dev;
  }
#endif
  return pdl_launch(PDL_MISC, k_pcg_control, 1, 1, 0, st, pq, rr, tol_nb2, out, pause, guard, seq);
}

__global__ void k_pcg_control_graph(const double* pq, const double* rr, const double* tol_nb2, double* out,
                                    int* pause, int* ctl, cudaGraphConditionalHandle cond) {
  pdl_trigger();
  pdl_wait();
  volatile int* vctl = ctl;
  if (*reinterpret_cast<volatile int*>(pause)) {  // an earlier iteration of this body stopped
    cudaGraphSetConditional(cond, 0);
    return;
  }
  const int it = vctl[1] + 1;
  vctl[1] = it;
  const double p = *pq, r2 = *rr;
  const bool bad = !isfinite(p) || p <= 0.0 || !isfinite(r2);
  // slightly looser than the host's |r| <= tol |b| (see k_pcg_control)
  const bool stop = bad || r2 <= *tol_nb2 * (1.0 + 1e-12);
  volatile double* o = out + 4 * (it & 1);
  o[0] = p;
  o[1] = r2;
  o[2] = stop ? 1.0 : 0.0;
  if (stop || it >= vctl[2]) {
    *reinterpret_cast<volatile int*>(pause) = 1;  // the rest of the body exits at its guards
    cudaGraphSetConditional(cond, 0);
    volatile double* rep = out + 8;
    rep[0] = p;
    rep[1] = r2;
    rep[2] = stop ? 1.0 : 0.0;
    __threadfence_system();
    rep[3] = (double)it;
  }
}

__global__ void k_pcg_graph_prep(int* ctl, int it0m1, int max_inner, double* tol_slot, double tol_nb2) {
  ctl[1] = it0m1;
  ctl[2] = max_inner;
  *tol_slot = tol_nb2;
}

cudaError_t launch_pcg_control_graph(cudaStream_t st, LaunchCounter* lc, const double* pq, const double* rr,
                                     const double* tol_nb2, double* out, int* pause, int* ctl,
                                     cudaGraphConditionalHandle cond) {
  count(lc);
  return pdl_launch(PDL_MISC, k_pcg_control_graph, 1, 1, 0, st, pq, rr, tol_nb2, out, pause, ctl, cond);
}

cudaError_t launch_pcg_graph_prep(cudaStream_t st, LaunchCounter* lc, int* ctl, int it0m1, int max_inner,
                                  double* tol_slot, double tol_nb2) {
  count(lc);
  k_pcg_graph_prep<<<1, 1, 0, st>>>(ctl, it0m1, max_inner, tol_slot, tol_nb2);
  return cudaGetLastError();
}

namespace {
thread_local bool t_pdl_off = false;
}
bool pdl_suspended() { return t_pdl_off; }
void pdl_suspend(bool on) { t_pdl_off = on; }

bool pdl_after(bool l1) {
  thread_local bool last_l1 = false;
  const bool ok = !l1 || last_l1;
  last_l1 = l1;
  return ok;
}

// Default: every class except the K row passes (launched behind a column or
// preconditioner pass they measure faster without PDL: C2 891 -> 870 us per
// iteration, C3 2158 -> 2124, C4 9746 -> 9712, C1 unchanged).
int pdl_mask() {
  static const int m = [] {
    const char* e = std::getenv("FDG_PDL_MASK");
    return e ? std::atoi(e) : ~(int)PDL_KROW;
  }();
  return m;
}

cudaError_t launch_copy(cudaStream_t st, LaunchCounter* lc, double* dst, const double* src, size_t N) {
  count(lc);
  k_copy<<<ew_grid(N), EW_THREADS, 0, st>>>(dst, src, N);
  return cudaGetLastError();
}
cudaError_t launch_fill(cudaStream_t st, LaunchCounter* lc, double* dst, double v, size_t N) {
  count(lc);
  k_fill<<<ew_grid(N), EW_THREADS, 0, st>>>(dst, v, N);
  return cudaGetLastError();
}
cudaError_t launch_any_nonzero(cudaStream_t st, LaunchCounter* lc, const double* x, size_t N, int* flag) {
  count(lc);
  k_any_nonzero<<<ew_grid(N), EW_THREADS, 0, st>>>(x, N, flag);
  return cudaGetLastError();
}
// |a|^2 and |b|^2 in one pass, into red.result[0], red.result[1]
__global__ void k_norms2(const double* a, const double* b, size_t N, RedSlot red) {
  __shared__ double scratch[64];
  double sa = 0.0, sb = 0.0;
  GRID_STRIDE(i, N) {
    const double u = a[i], v = b[i];
    sa += u * u;
    sb += v * v;
  }
  double vv[2] = {sa, sb};
  block_reduce<RED_SUM, 2>(vv, scratch);
  grid_finalize<RED_SUM, 2>(vv, red, scratch);
}
cudaError_t launch_norms2(cudaStream_t st, LaunchCounter* lc, const double* a, const double* b, size_t N,
                          RedSlot red) {
  count(lc);
  k_norms2<<<ew_grid(N), EW_THREADS, 0, st>>>(a, b, N, red);
  return cudaGetLastError();
}
cudaError_t launch_dot(cudaStream_t st, LaunchCounter* lc, const double* a, const double* b, size_t N,
                       RedSlot red) {
  count(lc);
  k_dot<<<ew_grid(N), EW_THREADS, 0, st>>>(a, b, N, red);
  return cudaGetLastError();
}
cudaError_t launch_cg_update(cudaStream_t st, LaunchCounter* lc, double* x, double* p, const double* z, size_t N,
                             const double* a_num, const double* a_den, const double* b_num, const double* b_den,
                             bool update_x) {
  count(lc);
  k_cg_update<<<ew_grid(N), EW_THREADS, 0, st>>>(x, p, z, N, a_num, a_den, b_num, b_den, update_x ? 1 : 0);
  return cudaGetLastError();
}
cudaError_t launch_axpy_dev(cudaStream_t st, LaunchCounter* lc, double* x, const double* p, size_t N,
                            const double* a_num, const double* a_den, const int* guard) {
  count(lc);
  return pdl_launch(PDL_MISC, k_axpy_dev, ew_grid(N), EW_THREADS, 0, st, x, p, N, a_num, a_den, guard);
}
cudaError_t launch_residual(cudaStream_t st, LaunchCounter* lc, double* r, const double* b, const double* q,
                            size_t N, RedSlot red) {
  count(lc);
  k_residual<<<ew_grid(N), EW_THREADS, 0, st>>>(r, b, q, N, red);
  return cudaGetLastError();
}
cudaError_t launch_scale_by_slice(cudaStream_t st, LaunchCounter* lc, double* out, const double* x,
                                  const double* coef, size_t slice, size_t N) {
  count(lc);
  k_scale_by_slice<<<ew_grid(N), EW_THREADS, 0, st>>>(out, x, coef, slice, N);
  return cudaGetLastError();
}
cudaError_t launch_rhs_pre(cudaStream_t st, LaunchCounter* lc, const AdmmScalars& a, const double* p,
                           const double* w_v, const double* z_v, const double* a2inv, const double* m2,
                           double* r_cache, double* tmp, size_t slice, size_t N) {
  count(lc);
  k_rhs_pre<<<ew_grid(N), EW_THREADS, 0, st>>>(a, p, w_v, z_v, a2inv, m2, r_cache, tmp, slice, N);
  return cudaGetLastError();
}
cudaError_t launch_rhs_post(cudaStream_t st, LaunchCounter* lc, const AdmmScalars& a, double* rhs,
                            const double* ybar, const double* w_y, const double* z_y, const double* diag_j,
                            size_t slice, size_t N) {
  count(lc);
  k_rhs_post<<<ew_grid(N), EW_THREADS, 0, st>>>(a, rhs, ybar, w_y, z_y, diag_j, slice, N);
  return cudaGetLastError();
}
cudaError_t launch_admm_update(cudaStream_t st, LaunchCounter* lc, const AdmmScalars& a, const double* y,
                               double* v, double* z_y, double* z_v, double* p, double* w_y, double* w_v,
                               const double* By, const double* r_cache, const double* a2inv, const double* m2,
                               size_t slice, size_t N, RedSlot red) {
  count(lc);
  k_admm_update<<<ew_grid(N), EW_THREADS, 0, st>>>(a, y, v, z_y, z_v, p, w_y, w_v, By, r_cache, a2inv, m2,
                                                   slice, N, red);
  return cudaGetLastError();
}
cudaError_t launch_dual_inf(cudaStream_t st, LaunchCounter* lc, const double* y, const double* ybar,
                            const double* btp, const double* w_y, const double* v, const double* p,
                            const double* w_v, const double* diag_j, const double* diag_j2, size_t slice,
                            size_t N, RedSlot red) {
  count(lc);
  k_dual_inf<<<ew_grid(N), EW_THREADS, 0, st>>>(y, ybar, btp, w_y, v, p, w_v, diag_j, diag_j2, slice, N, red);
  return cudaGetLastError();
}
cudaError_t launch_objective(cudaStream_t st, LaunchCounter* lc, const double* y, const double* ybar,
                             const double* v, const double* diag_j, const double* diag_j2, size_t slice,
                             size_t N, RedSlot red) {
  count(lc);
  k_objective<<<ew_grid(N), EW_THREADS, 0, st>>>(y, ybar, v, diag_j, diag_j2, slice, N, red);
  return cudaGetLastError();
}

// ============================================================== Bluestein
// Non-power-of-two Hartley transforms of the 2-level spatial preconditioner
// (BASELINE C1, fdg_api.cu pc2_apply_dev).  Z = DFT_n(a + ib) by Bluestein,
//   Z_k = conj(c_k) sum_j c_{k-j} conj(c_j) z_j,   c_m = exp(i pi m^2 / n),
// i.e. a chirp pre-multiply, a Toeplitz convolution with the chirp (the
// row / column pass kernels with a complex symbol) and a chirp post-multiply;
// the Hartley transforms of a and b follow from Z_k and Z_{n-k}
// (fdg_fft.cuh hartley_split).  Real fibres travel in pairs: rows 2q, 2q+1
// (x2 stage, row pitch n2) or columns 2p, 2p+1 (x1 stage, row pitch P2 =
// n2 rounded up to even) are the real and imaginary parts of one lane.
namespace {
__device__ __forceinline__ double2 ld_pair(const double* p) { return *reinterpret_cast<const double2*>(p); }
}  // namespace

// x2 pre: out[2q][k] + i out[2q+1][k] = (in[2q][k] + i in[2q+1][k]) conj(c2[k])
__global__ void k_bs_pre_rows(const double* in, double* out, long F, int n2, const double2* c2) {
  const long Q = (F + 1) / 2;
  GRID_STRIDE(e, (size_t)Q * n2) {
    const long q = (long)(e / n2);
    const int k = (int)(e - (size_t)q * n2);
    const long f0 = 2 * q, f1 = 2 * q + 1;
    const double a = in[f0 * n2 + k], b = f1 < F ? in[f1 * n2 + k] : 0.0;
    const double2 z = cmulc(make_double2(a, b), c2[k]);
    out[f0 * n2 + k] = z.x;
    out[f1 * n2 + k] = z.y;
  }
}

// x2 post (forward) + x1 pre: v [Fp][n2] -> u [nt][n1][P2]
__global__ void k_bs_rows_to_cols(const double* v, double* u, long F, int n1, int n2, int P2, const double2* c2,
                                  const double2* c1) {
  const long Q = (F + 1) / 2;
  const int Pp = P2 / 2;
  GRID_STRIDE(e, (size_t)Q * Pp) {
    const long q = (long)(e / Pp);
    const int p = (int)(e - (size_t)q * Pp);
    const double* r0 = v + 2 * q * n2;
    const double* r1 = r0 + n2;
    double2 h[2];  // h[j] = (row 2q, row 2q+1) Hartley values at column 2p + j
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int k = 2 * p + j;
      if (k < n2) {
        const int km = k == 0 ? 0 : n2 - k;
        const double2 Z = cmulc(make_double2(r0[k], r1[k]), c2[k]);
        const double2 Zm = cmulc(make_double2(r0[km], r1[km]), c2[km]);
        h[j] = hartley_split(Z, Zm);
      } else {
        h[j] = make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const long f = 2 * q + s;
      if (f >= F) break;
      const long o = f / n1;
      const int i = (int)(f - o * n1);
      const double2 z = s ? make_double2(h[0].y, h[1].y) : make_double2(h[0].x, h[1].x);
      const double2 w = cmulc(z, c1[i]);
      *reinterpret_cast<double2*>(u + (o * n1 + i) * P2 + 2 * p) = w;
    }
  }
}

// x1 post (forward) + 1/(lam1[i] + lam2[j]) + x1 pre (inverse): [nt][n1][P2] -> same
__global__ void k_bs_cols_filter(const double* v, double* u, int nt, int n1, int n2, int P2, const double2* c1,
                                 const double* lam1, const double* lam2) {
  const int Pp = P2 / 2;
  GRID_STRIDE(e, (size_t)nt * n1 * Pp) {
    const long row = (long)(e / Pp);  // o * n1 + i
    const int p = (int)(e - (size_t)row * Pp);
    const long o = row / n1;
    const int i = (int)(row - o * n1);
    const int im = i == 0 ? 0 : n1 - i;
    const double2 Z = cmulc(ld_pair(v + row * P2 + 2 * p), c1[i]);
    const double2 Zm = cmulc(ld_pair(v + (o * n1 + im) * P2 + 2 * p), c1[im]);
    double2 h = hartley_split(Z, Zm);
    h.x /= lam1[i] + lam2[2 * p];
    h.y = 2 * p + 1 < n2 ? h.y / (lam1[i] + lam2[2 * p + 1]) : 0.0;
    *reinterpret_cast<double2*>(u + row * P2 + 2 * p) = cmulc(h, c1[i]);
  }
}

// x1 post (inverse) + x2 pre (inverse): v [nt][n1][P2] -> u [Fp][n2]
__global__ void k_bs_cols_to_rows(const double* v, double* u, long F, int n1, int n2, int P2, const double2* c1,
                                  const double2* c2) {
  const long Q = (F + 1) / 2;
  const int Pp = P2 / 2;
  GRID_STRIDE(e, (size_t)Q * Pp) {
    const long q = (long)(e / Pp);
    const int p = (int)(e - (size_t)q * Pp);
    double2 h[2];  // h[s] = (column 2p, column 2p+1) Hartley values of row 2q + s
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const long f = 2 * q + s;
      if (f < F) {
        const long o = f / n1;
        const int i = (int)(f - o * n1);
        const int im = i == 0 ? 0 : n1 - i;
        const double2 Z = cmulc(ld_pair(v + f * P2 + 2 * p), c1[i]);
        const double2 Zm = cmulc(ld_pair(v + (o * n1 + im) * P2 + 2 * p), c1[im]);
        h[s] = hartley_split(Z, Zm);
      } else {
        h[s] = make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int k = 2 * p + j;
      if (k >= n2) break;
      const double2 z = j ? make_double2(h[0].y, h[1].y) : make_double2(h[0].x, h[1].x);
      const double2 w = cmulc(z, c2[k]);
      u[2 * q * n2 + k] = w.x;
      u[(2 * q + 1) * n2 + k] = w.y;
    }
  }
}

// x2 post (inverse) + scale: v [Fp][n2] -> z [F][n2]
__global__ void k_bs_post_rows(const double* v, double* z, long F, int n2, const double2* c2, double scale) {
  const long Q = (F + 1) / 2;
  GRID_STRIDE(e, (size_t)Q * n2) {
    const long q = (long)(e / n2);
    const int k = (int)(e - (size_t)q * n2);
    const int km = k == 0 ? 0 : n2 - k;
    const double* r0 = v + 2 * q * n2;
    const double* r1 = r0 + n2;
    const double2 Z = cmulc(make_double2(r0[k], r1[k]), c2[k]);
    const double2 Zm = cmulc(make_double2(r0[km], r1[km]), c2[km]);
    const double2 h = hartley_split(Z, Zm);
    z[2 * q * n2 + k] = scale * h.x;
    if (2 * q + 1 < F) z[(2 * q + 1) * n2 + k] = scale * h.y;
  }
}

cudaError_t launch_bs_pre_rows(cudaStream_t st, LaunchCounter* lc, const double* in, double* out, long F, int n2,
                               const double2* c2) {
  count(lc);
  k_bs_pre_rows<<<ew_grid((size_t)((F + 1) / 2) * n2), EW_THREADS, 0, st>>>(in, out, F, n2, c2);
  return cudaGetLastError();
}
cudaError_t launch_bs_rows_to_cols(cudaStream_t st, LaunchCounter* lc, const double* v, double* u, long F, int n1,
                                   int n2, int P2, const double2* c2, const double2* c1) {
  count(lc);
  k_bs_rows_to_cols<<<ew_grid((size_t)((F + 1) / 2) * (P2 / 2)), EW_THREADS, 0, st>>>(v, u, F, n1, n2, P2, c2, c1);
  return cudaGetLastError();
}
cudaError_t launch_bs_cols_filter(cudaStream_t st, LaunchCounter* lc, const double* v, double* u, int nt, int n1,
                                  int n2, int P2, const double2* c1, const double* lam1, const double* lam2) {
  count(lc);
  k_bs_cols_filter<<<ew_grid((size_t)nt * n1 * (P2 / 2)), EW_THREADS, 0, st>>>(v, u, nt, n1, n2, P2, c1, lam1, lam2);
  return cudaGetLastError();
}
cudaError_t launch_bs_cols_to_rows(cudaStream_t st, LaunchCounter* lc, const double* v, double* u, long F, int n1,
                                   int n2, int P2, const double2* c1, const double2* c2) {
  count(lc);
  k_bs_cols_to_rows<<<ew_grid((size_t)((F + 1) / 2) * (P2 / 2)), EW_THREADS, 0, st>>>(v, u, F, n1, n2, P2, c1, c2);
  return cudaGetLastError();
}
cudaError_t launch_bs_post_rows(cudaStream_t st, LaunchCounter* lc, const double* v, double* z, long F, int n2,
                                const double2* c2, double scale) {
  count(lc);
  k_bs_post_rows<<<ew_grid((size_t)((F + 1) / 2) * n2), EW_THREADS, 0, st>>>(v, z, F, n2, c2, scale);
  return cudaGetLastError();
}

bool encode_col_map(CUtensorMap* map, const double* base, long rows, int C, int W, int brows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return false;
  const cuuint64_t gdim[2] = {(cuuint64_t)C, (cuuint64_t)rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)C * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)brows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), gdim, gstride, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t max_partials_needed(int nt, int n1, int n2) {
  // Row/column/Hartley grids use >= 2*4 fibres per CTA; elementwise grids are
  // capped at 148*8 CTAs.
  auto cdiv = [](size_t a, size_t b) { return (a + b - 1) / b; };
  size_t m = 148 * 8;
  m = std::max(m, cdiv((size_t)nt * n1, 8));       // row passes
  m = std::max(m, (size_t)nt * cdiv(n2, 8));       // x1 column passes
  m = std::max(m, cdiv((size_t)n1 * n2, 8));       // t passes
  return m + 1;
}

}  // namespace fdg
