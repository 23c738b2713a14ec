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
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "fdg_fft.cuh"
#include "fdg_internal.h"
#include "fdg_reduce.cuh"

namespace fdg {

// ------------------------------------------------------------ tile configs
template <int L>
struct Cfg {
  static constexpr int R = L <= 8 ? L : (L <= 512 ? 8 : 16);
  static constexpr int T = L / R;
  static constexpr int G0 = L >= 2048 ? 4 : 8;
  static constexpr int G = (G0 * T < 32) ? (32 / T) : G0;
  static constexpr int THREADS = G * T;
  static constexpr size_t SMEM = (size_t)L * G * sizeof(double2);
};

__device__ __forceinline__ size_t idx2(size_t a, size_t b, size_t n) { return a * n + b; }

// =================================================================== rows
// Row pass along x2 (contiguous fibres of length n; embedding length L).
//   MODE 0 (apply):  out = psi*time(x) + scale * T2 x
//   MODE 1 (S out):  q = vp + psi*time^T(x) + scale * T2 x; q_out = q (opt);
//                    r -= (num/den) q; reduce |r|^2
struct RowArgs {
  const double* x;
  const double* vp;
  double* out;
  double* q_out;
  double* r;
  int nt, n1, n;
  const double2* sym;
  const double2* tw;
  double scale;
  int tkind;  // 1: stencil
  double tc0, tc1;
  int tdir;  // -1: uses k-1 (forward B), +1: uses k+1 (adjoint)
  const double* a_num;
  const double* a_den;
  RedSlot red;
};

template <int L, int MODE>
__global__ void __launch_bounds__(Cfg<L>::THREADS) k_row(RowArgs a) {
  using C = Cfg<L>;
  constexpr int R = C::R, T = C::T, G = C::G, H = (R + 1) / 2;
  extern __shared__ double2 sm[];
  __shared__ double scratch[32];
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  const long F = (long)a.nt * a.n1;
  const long f = ((long)blockIdx.x * G + g) * 2;
  const bool va = f < F, vb = f + 1 < F;
  const int n = a.n;
  double2 v[R];
  double2 xr[H];
#pragma unroll
  for (int m = 0; m < R; ++m) {
    const int pos = t + m * T;
    double2 z = make_double2(0.0, 0.0);
    if (m < H && pos < n) {
      if (va) z.x = __ldg(&a.x[idx2(f, pos, n)]);
      if (vb) z.y = __ldg(&a.x[idx2(f + 1, pos, n)]);
    }
    v[m] = z;
    if (m < H) xr[m] = z;
  }
  fft_lane<L, R, G, false>(v, sm, t, g, a.tw);
#pragma unroll
  for (int m = 0; m < R; ++m) v[m] = cmul(v[m], __ldg(&a.sym[t + m * T]));
  fft_lane<L, R, G, true>(v, sm, t, g, a.tw);

  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < H; ++m) {
    const int pos = t + m * T;
    if (pos >= n) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const long fh = f + h;
      if (fh >= F) continue;
      const double xv = h ? xr[m].y : xr[m].x;
      const double tv = h ? v[m].y : v[m].x;
      double val = a.scale * tv;
      if (a.tkind == 1) {
        const int k = (int)(fh / a.n1);
        double nb = 0.0;
        if (a.tdir < 0 && k >= 1) nb = __ldg(&a.x[idx2(fh - a.n1, pos, n)]);
        if (a.tdir > 0 && k + 1 < a.nt) nb = __ldg(&a.x[idx2(fh + a.n1, pos, n)]);
        val += a.tc0 * xv + a.tc1 * nb;
      }
      const size_t o = idx2(fh, pos, n);
      if constexpr (MODE == 0) {
        a.out[o] = val;
      } else {
        const double q = __ldg(&a.vp[o]) + val;
        if (a.q_out) a.q_out[o] = q;
        if (a.r) {
          const double alpha = *a.a_num / *a.a_den;
          const double rn = a.r[o] - alpha * q;
          a.r[o] = rn;
          acc += rn * rn;
        }
      }
    }
  }
  if constexpr (MODE == 1) {
    if (a.r) {
      double vv[1] = {acc};
      block_reduce<RED_SUM, 1>(vv, scratch);
      grid_finalize<RED_SUM, 1>(vv, a.red, scratch);
    }
  }
}

// ================================================================ columns
// Column pass along an axis of length n with inner stride C, outer count O:
// element (o, pos, c) at o*n*C + pos*C + c.
//   MODE 0 (acc): out = acc + scale * T x            (acc may alias out)
//   MODE 2 (S mid, axis x1): Bp = u + scale*T p; w = Bp * inv_m2[o];
//        vp = scale * T w + a1[o] p; reduce sum(a1 p^2 + w Bp)
struct ColArgs {
  const double* x;
  const double* acc;
  double* out;
  double* w;
  int O, n, C;
  const double2* sym;
  const double2* tw;
  double scale;
  const double* inv_m2;
  const double* a1;
  RedSlot red;
};

template <int L>
__device__ __forceinline__ void col_load(const double* __restrict__ base, int n, int C, long c, int t,
                                         double2 (&v)[Cfg<L>::R], int H) {
  constexpr int R = Cfg<L>::R, T = Cfg<L>::T;
  const bool pair = (c + 1 < C) && ((C & 1) == 0);
#pragma unroll
  for (int m = 0; m < R; ++m) {
    const int pos = t + m * T;
    double2 z = make_double2(0.0, 0.0);
    if (m < H && pos < n && c < C) {
      const double* p = base + (size_t)pos * C + c;
      if (pair) {
        z = __ldg(reinterpret_cast<const double2*>(p));
      } else {
        z.x = __ldg(p);
        if (c + 1 < C) z.y = __ldg(p + 1);
      }
    }
    v[m] = z;
  }
}

__device__ __forceinline__ void col_store(double* base, int pos, int C, long c, double2 val) {
  double* p = base + (size_t)pos * C + c;
  if ((c + 1 < C) && ((C & 1) == 0)) {
    *reinterpret_cast<double2*>(p) = val;
  } else {
    p[0] = val.x;
    if (c + 1 < C) p[1] = val.y;
  }
}

template <int L, int MODE>
__global__ void __launch_bounds__(Cfg<L>::THREADS) k_col(ColArgs a) {
  using Cf = Cfg<L>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G, H = (R + 1) / 2;
  extern __shared__ double2 sm[];
  __shared__ double scratch[32];
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  const int o = blockIdx.y;
  const long c = ((long)blockIdx.x * G + g) * 2;
  const int n = a.n, C = a.C;
  const size_t base = (size_t)o * n * C;
  double2 v[R];
  double2 keep[H];
  col_load<L>(a.x + base, n, C, c, t, v, H);
#pragma unroll
  for (int m = 0; m < H; ++m) keep[m] = v[m];
  fft_lane<L, R, G, false>(v, sm, t, g, a.tw);
#pragma unroll
  for (int m = 0; m < R; ++m) v[m] = cmul(v[m], __ldg(&a.sym[t + m * T]));
  fft_lane<L, R, G, true>(v, sm, t, g, a.tw);

  if constexpr (MODE == 0) {
#pragma unroll
    for (int m = 0; m < H; ++m) {
      const int pos = t + m * T;
      if (pos >= n || c >= C) continue;
      double2 acc = make_double2(0.0, 0.0);
      if (a.acc) {
        const double* p = a.acc + base + (size_t)pos * C + c;
        acc.x = p[0];
        if (c + 1 < C) acc.y = p[1];
      }
      col_store(a.out + base, pos, C, c, make_double2(acc.x + a.scale * v[m].x, acc.y + a.scale * v[m].y));
    }
  } else {
    // S mid pass: u is a.acc, w -> a.w, vp -> a.out
    const double im2 = a.inv_m2[o], a1 = a.a1[o];
    double e = 0.0;
    double2 u[H];
    double2 zero2 = make_double2(0.0, 0.0);
#pragma unroll
    for (int m = 0; m < H; ++m) {
      const int pos = t + m * T;
      u[m] = zero2;
      if (pos < n && c < C) {
        const double* p = a.acc + base + (size_t)pos * C + c;
        u[m].x = p[0];
        if (c + 1 < C) u[m].y = p[1];
      }
    }
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int pos = t + m * T;
      if (m < H && pos < n && c < C) {
        const double bx = u[m].x + a.scale * v[m].x;
        const double by = u[m].y + a.scale * v[m].y;
        const double wx = bx * im2, wy = (c + 1 < C) ? by * im2 : 0.0;
        e += a1 * keep[m].x * keep[m].x + wx * bx;
        if (c + 1 < C) e += a1 * keep[m].y * keep[m].y + wy * by;
        col_store(a.w + base, pos, C, c, make_double2(wx, wy));
        v[m] = make_double2(wx, wy);
      } else {
        v[m] = zero2;
      }
    }
    fft_lane<L, R, G, false>(v, sm, t, g, a.tw);
#pragma unroll
    for (int m = 0; m < R; ++m) v[m] = cmul(v[m], __ldg(&a.sym[t + m * T]));
    fft_lane<L, R, G, true>(v, sm, t, g, a.tw);
#pragma unroll
    for (int m = 0; m < H; ++m) {
      const int pos = t + m * T;
      if (pos >= n || c >= C) continue;
      col_store(a.out + base, pos, C, c,
                make_double2(a.scale * v[m].x + a1 * keep[m].x, a.scale * v[m].y + a1 * keep[m].y));
    }
    double vv[1] = {e};
    block_reduce<RED_SUM, 1>(vv, scratch);
    grid_finalize<RED_SUM, 1>(vv, a.red, scratch);
  }
}

// ============================================================== Hartley
// Real Hartley transform H[f] = sum_j x_j cas(2 pi j f / N) of two real
// fibres packed as a + i b into one complex FFT (fdg_fft.cuh hartley_split).
// For the circulant preconditioner the multiplier lambda_S is even in every
// axis (spatial T. Chan eigenvalues are real and even; |conj(l_t) - s| =
// |l_t - s| for real s), so F^-1 D F == H^-1 D H axis by axis: all three
// passes stay real (N doubles in, N doubles out), see DESIGN.md.
template <int N>
__global__ void __launch_bounds__(Cfg<N>::THREADS) k_hartley_row(const double* in, double* out, int F,
                                                                 const double2* tw, const double* rdot,
                                                                 RedSlot red) {
  using Cf = Cfg<N>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G;
  extern __shared__ double2 sm[];
  __shared__ double scratch[32];
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  const long f = ((long)blockIdx.x * G + g) * 2;
  const bool va = f < F, vb = f + 1 < F;
  double2 v[R], w[R];
#pragma unroll
  for (int m = 0; m < R; ++m) {
    const int pos = t + m * T;
    v[m].x = va ? __ldg(&in[idx2(f, pos, N)]) : 0.0;
    v[m].y = vb ? __ldg(&in[idx2(f + 1, pos, N)]) : 0.0;
  }
  fft_lane<N, R, G, false>(v, sm, t, g, tw);
  mirror_lane<N, R, G>(v, w, sm, t, g);
  double acc = 0.0;
#pragma unroll
  for (int m = 0; m < R; ++m) {
    const int pos = t + m * T;
    const double2 h = hartley_split(v[m], w[m]);
    if (va) {
      out[idx2(f, pos, N)] = h.x;
      if (rdot) acc += __ldg(&rdot[idx2(f, pos, N)]) * h.x;
    }
    if (vb) {
      out[idx2(f + 1, pos, N)] = h.y;
      if (rdot) acc += __ldg(&rdot[idx2(f + 1, pos, N)]) * h.y;
    }
  }
  if (rdot) {
    double vv[1] = {acc};
    block_reduce<RED_SUM, 1>(vv, scratch);
    grid_finalize<RED_SUM, 1>(vv, red, scratch);
  }
}

template <int N>
__global__ void __launch_bounds__(Cfg<N>::THREADS) k_hartley_col(double* data, int C, const double2* tw) {
  using Cf = Cfg<N>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G;
  extern __shared__ double2 sm[];
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  const long c = ((long)blockIdx.x * G + g) * 2;
  const size_t base = (size_t)blockIdx.y * N * C;
  double2 v[R], w[R];
  col_load<N>(data + base, N, C, c, t, v, R);
  fft_lane<N, R, G, false>(v, sm, t, g, tw);
  mirror_lane<N, R, G>(v, w, sm, t, g);
#pragma unroll
  for (int m = 0; m < R; ++m) {
    const int pos = t + m * T;
    if (c < C) col_store(data + base, pos, C, c, hartley_split(v[m], w[m]));
  }
}

// t pass of the preconditioner: Hartley along t, divide by lambda_S (computed
// in registers from the 1-D eigenvalues, circulant.cpp:28-41, 76-90) and by
// N (circulant.cpp:62-64), Hartley along t again.
template <int N>
__global__ void __launch_bounds__(Cfg<N>::THREADS) k_t_filter(double* data, PcTables pt) {
  using Cf = Cfg<N>;
  constexpr int R = Cf::R, T = Cf::T, G = Cf::G;
  extern __shared__ double2 sm[];
  const int g = threadIdx.x % G, t = threadIdx.x / G;
  const int C = pt.n1 * pt.n2;
  const long c = ((long)blockIdx.x * G + g) * 2;
  double2 v[R], w[R];
  col_load<N>(data, N, C, c, t, v, R);
  fft_lane<N, R, G, false>(v, sm, t, g, pt.tw_t);
  mirror_lane<N, R, G>(v, w, sm, t, g);
  // spatial eigenvalue sums of the two packed columns
  double2 sa = make_double2(0.0, 0.0), sb = make_double2(0.0, 0.0);
  if (c < C) {
    const int i = (int)(c / pt.n2), j = (int)(c % pt.n2);
    const double2 l1 = __ldg(&pt.lam_1[i]), l2 = __ldg(&pt.lam_2[j]);
    sa = make_double2(l1.x + l2.x, l1.y + l2.y);
  }
  if (c + 1 < C) {
    const int i = (int)((c + 1) / pt.n2), j = (int)((c + 1) % pt.n2);
    const double2 l1 = __ldg(&pt.lam_1[i]), l2 = __ldg(&pt.lam_2[j]);
    sb = make_double2(l1.x + l2.x, l1.y + l2.y);
  }
#pragma unroll
  for (int m = 0; m < R; ++m) {
    const int k = t + m * T;
    const double2 h = hartley_split(v[m], w[m]);
    const double2 lt = __ldg(&pt.lam_t[k]);
    const double bax = pt.psi * (lt.x - sa.x), bay = pt.psi * (lt.y - sa.y);
    const double bbx = pt.psi * (lt.x - sb.x), bby = pt.psi * (lt.y - sb.y);
    const double lsa = pt.base + (bax * bax + bay * bay) * pt.inv_m2;
    const double lsb = pt.base + (bbx * bbx + bby * bby) * pt.inv_m2;
    v[m] = make_double2(h.x / lsa * pt.inv_total, h.y / lsb * pt.inv_total);
  }
  fft_lane<N, R, G, false>(v, sm, t, g, pt.tw_t);
  mirror_lane<N, R, G>(v, w, sm, t, g);
#pragma unroll
  for (int m = 0; m < R; ++m) {
    const int pos = t + m * T;
    if (c < C) col_store(data, pos, C, c, hartley_split(v[m], w[m]));
  }
}

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
__global__ void k_axpy_dev(double* x, const double* p, size_t N, const double* an, const double* ad) {
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
#define FDG_POW2_CASES(X) X(2) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048)

// Opt in to > 48 KB dynamic shared memory once per kernel instantiation.
template <auto K>
static cudaError_t prep(size_t smem) {
  static int done_device = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_device != dev && smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  done_device = dev;
  return cudaSuccess;
}

static inline void count(LaunchCounter* lc, unsigned long long k = 1) {
  if (lc) lc->count += k;
}

static int pow2_ceil(long v) {
  int L = 1;
  while (L < v) L <<= 1;
  return L;
}

template <int L, int MODE>
static cudaError_t run_row(cudaStream_t st, const RowArgs& a) {
  using Cf = Cfg<L>;
  const long F = (long)a.nt * a.n1;
  const unsigned grid = (unsigned)((F + 2 * Cf::G - 1) / (2 * Cf::G));
  cudaError_t e = prep<k_row<L, MODE>>(Cf::SMEM);
  if (e != cudaSuccess) return e;
  k_row<L, MODE><<<grid, Cf::THREADS, Cf::SMEM, st>>>(a);
  return cudaGetLastError();
}

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

template <int L, int MODE>
static cudaError_t run_col(cudaStream_t st, const ColArgs& a) {
  using Cf = Cfg<L>;
  dim3 grid((unsigned)((a.C + 2 * Cf::G - 1) / (2 * Cf::G)), (unsigned)a.O);
  cudaError_t e = prep<k_col<L, MODE>>(Cf::SMEM);
  if (e != cudaSuccess) return e;
  k_col<L, MODE><<<grid, Cf::THREADS, Cf::SMEM, st>>>(a);
  return cudaGetLastError();
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
                             bool adjoint) {
  RowArgs a{};
  a.x = x;
  a.out = out;
  a.nt = nt;
  a.n1 = n1;
  a.n = n2;
  a.sym = s2.sym;
  a.tw = s2.tw;
  a.scale = scale;
  a.tkind = tf.kind == 1 ? 1 : 0;
  a.tc0 = psi * tf.c0;
  a.tc1 = psi * tf.c1;
  a.tdir = adjoint ? +1 : -1;
  count(lc);
  return dispatch_row<0>(st, s2.L, a);
}

cudaError_t launch_row_s_out(cudaStream_t st, LaunchCounter* lc, const double* w, const double* vp, double* q_out,
                             double* r, int nt, int n1, int n2, const AxisSym& s2, double scale,
                             const TimeFactor& tf, double psi, const double* alpha_num, const double* alpha_den,
                             RedSlot red) {
  RowArgs a{};
  a.x = w;
  a.vp = vp;
  a.q_out = q_out;
  a.r = r;
  a.nt = nt;
  a.n1 = n1;
  a.n = n2;
  a.sym = s2.sym;
  a.tw = s2.tw;
  a.scale = scale;
  a.tkind = tf.kind == 1 ? 1 : 0;
  a.tc0 = psi * tf.c0;
  a.tc1 = psi * tf.c1;
  a.tdir = +1;
  a.a_num = alpha_num;
  a.a_den = alpha_den;
  a.red = red;
  count(lc);
  return dispatch_row<1>(st, s2.L, a);
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
  a.tw = s.tw;
  a.scale = scale;
  count(lc);
  return dispatch_col<0>(st, s.L, a);
}

cudaError_t launch_col_s_mid(cudaStream_t st, LaunchCounter* lc, const double* p, const double* u, double* w,
                             double* vp, int nt, int n1, int n2, const AxisSym& s1, double scale,
                             const double* inv_m2, const double* a1, RedSlot red) {
  ColArgs a{};
  a.x = p;
  a.acc = u;
  a.w = w;
  a.out = vp;
  a.O = nt;
  a.n = n1;
  a.C = n2;
  a.sym = s1.sym;
  a.tw = s1.tw;
  a.scale = scale;
  a.inv_m2 = inv_m2;
  a.a1 = a1;
  a.red = red;
  count(lc);
  return dispatch_col<2>(st, s1.L, a);
}

template <int N>
static cudaError_t run_hrow(cudaStream_t st, const double* in, double* out, int F, const double2* tw,
                            const double* rdot, RedSlot red) {
  using Cf = Cfg<N>;
  const unsigned grid = (unsigned)((F + 2 * Cf::G - 1) / (2 * Cf::G));
  cudaError_t e = prep<k_hartley_row<N>>(Cf::SMEM);
  if (e != cudaSuccess) return e;
  k_hartley_row<N><<<grid, Cf::THREADS, Cf::SMEM, st>>>(in, out, F, tw, rdot, red);
  return cudaGetLastError();
}

template <int N>
static cudaError_t run_hcol(cudaStream_t st, double* data, int O, int C, const double2* tw) {
  using Cf = Cfg<N>;
  dim3 grid((unsigned)((C + 2 * Cf::G - 1) / (2 * Cf::G)), (unsigned)O);
  cudaError_t e = prep<k_hartley_col<N>>(Cf::SMEM);
  if (e != cudaSuccess) return e;
  k_hartley_col<N><<<grid, Cf::THREADS, Cf::SMEM, st>>>(data, C, tw);
  return cudaGetLastError();
}

template <int N>
static cudaError_t run_tf(cudaStream_t st, double* data, const PcTables& pt) {
  using Cf = Cfg<N>;
  const long C = (long)pt.n1 * pt.n2;
  const unsigned grid = (unsigned)((C + 2 * Cf::G - 1) / (2 * Cf::G));
  cudaError_t e = prep<k_t_filter<N>>(Cf::SMEM);
  if (e != cudaSuccess) return e;
  k_t_filter<N><<<grid, Cf::THREADS, Cf::SMEM, st>>>(data, pt);
  return cudaGetLastError();
}

#define FDG_POW2_CASES1(X) X(1) FDG_POW2_CASES(X)

cudaError_t launch_hartley_row(cudaStream_t st, LaunchCounter* lc, const double* in, double* out, int F, int n,
                               const double2* tw, const double* rdot, RedSlot red) {
  count(lc);
  switch (n) {
#define X(NN) \
  case NN: return run_hrow<NN>(st, in, out, F, tw, rdot, red);
    FDG_POW2_CASES1(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_hartley_col(cudaStream_t st, LaunchCounter* lc, double* data, int O, int n, int C,
                               const double2* tw) {
  count(lc);
  switch (n) {
#define X(NN) \
  case NN: return run_hcol<NN>(st, data, O, C, tw);
    FDG_POW2_CASES1(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_t_filter(cudaStream_t st, LaunchCounter* lc, double* data, const PcTables& pt) {
  count(lc);
  switch (pt.nt) {
#define X(NN) \
  case NN: return run_tf<NN>(st, data, pt);
    FDG_POW2_CASES1(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
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
                            const double* a_num, const double* a_den) {
  count(lc);
  k_axpy_dev<<<ew_grid(N), EW_THREADS, 0, st>>>(x, p, N, a_num, a_den);
  return cudaGetLastError();
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
