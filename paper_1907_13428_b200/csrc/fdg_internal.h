// fdg_internal.h — host-side declarations shared by the C-ABI layer and the
// kernel launchers.  Not part of the public interface (include/fdg.h is).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "fdg_reduce.cuh"

namespace fdg {

// Device-resident description of one spatial/temporal Toeplitz factor used by
// the FFT passes: the full length-L circulant-embedding symbol (L pow2 >=
// 2n-1) and the matching twiddle table, both double2[L].
struct AxisSym {
  int n = 0;  // factor size
  int L = 0;  // embedding length (power of two)
  const double2* sym = nullptr;      // forward factor symbol
  const double2* sym_adj = nullptr;  // transposed factor symbol (== sym if symmetric)
  const double2* tw = nullptr;       // W_L twiddles
  const double2* twh = nullptr;      // per-pass twiddles of the L/2-point transform
  const double2* twist = nullptr;    // W_L^j, j < L/2 (split passes, fdg_conv.cuh)
  const double* sym_re = nullptr;      // real copy of sym when the factor is symmetric
  const double* sym_adj_re = nullptr;  // real copy of sym_adj
  const double2* tw256 = nullptr;      // Q-split passes (L >= 1024): 256-point plan
  const double2* twq = nullptr;        // Q-split passes: W_L^k, k < L
};

// Time coupling.  kind 0: no time term; 1: lower-bidiagonal stencil
// (c0 x_k + c1 x_{k-1}; adjoint c0 x_k + c1 x_{k+1}); 2: general Toeplitz
// applied by an FFT pass along t.
struct TimeFactor {
  int kind = 0;
  double c0 = 0.0, c1 = 0.0;  // unscaled stencil coefficients
  AxisSym fft;                // kind 2
};

// Per-launch bookkeeping (kernel count for the bench's gpu_launches claim).
struct LaunchCounter {
  unsigned long long count = 0;
};

// Spectral tables of the circulant preconditioner (1-D eigenvalues, complex).
struct PcTables {
  int nt = 0, n1 = 0, n2 = 0;
  const double2* lam_t = nullptr;
  const double2* lam_1 = nullptr;
  const double2* lam_2 = nullptr;
  const double2* tw_t = nullptr;  // W_nt
  const double2* tw_1 = nullptr;  // W_n1
  const double2* tw_2 = nullptr;  // W_n2
  double psi = 1.0, base = 0.0, inv_m2 = 0.0, inv_total = 0.0;
};

// ---------------------------------------------------------------- launchers
// All return cudaGetLastError() of the launch.  `lc` may be null.

// out = time(x) - psi * L2 x along x2 (rows), with time handled here when it
// is a stencil (kind 1).  adjoint selects the transposed time stencil.
cudaError_t launch_row_apply(cudaStream_t st, LaunchCounter* lc, const double* x, double* out, int nt,
                             int n1, int n2, const AxisSym& s2, double scale, const TimeFactor& tf,
                             double psi, bool adjoint,
                             const double2* chirp_in = nullptr);

// out = acc + scale * T(x) along an axis of length n with inner count C and
// outer count O (axis x1: O = nt, C = n2; axis t: O = 1, C = n1*n2).
cudaError_t launch_col_acc(cudaStream_t st, LaunchCounter* lc, const double* x, const double* acc,
                           double* out, int O, int n, int C, const AxisSym& s, double scale,
                           bool adjoint);

// Fused S pass 2 (x1 columns): Bp = u + scale*L1 p; w = Bp/m2[k];
// vp = scale*L1 w + a1[k] p; reduces sum(a1 p^2 + w Bp) = p^T S p.
cudaError_t launch_col_s_mid(cudaStream_t st, LaunchCounter* lc, const double* p, const double* u,
                             double* w, double* vp, int nt, int n1, int n2, const AxisSym& s1,
                             double scale, const double* inv_m2, const double* a1, RedSlot red,
                             const int* guard = nullptr);

// Fused S pass 3 (x2 rows) + residual update: q = vp + time^T(w) + scale*L2 w;
// if q_out: q_out = q; if r: r -= alpha q with alpha = *num / *den, reduce |r|^2.
cudaError_t launch_row_s_out(cudaStream_t st, LaunchCounter* lc, const double* w, const double* vp,
                             double* q_out, double* r, int nt, int n1, int n2, const AxisSym& s2,
                             double scale, const TimeFactor& tf, double psi, const double* alpha_num,
                             const double* alpha_den, RedSlot red, const int* guard = nullptr,
                             const double* r_in = nullptr);

// Fused CG update + B row pass (K9 folded into K1): d_new = z + beta d_old
// (beta = *b_num / *b_den; first: d_new = z), written to dnew and used as the
// FFT input; u = row(d_new) like launch_row_apply; if upd_x: x += alpha d_old
// (alpha = *a_num / *a_den).  Requires a bidiagonal or absent time factor.
cudaError_t launch_row_fused(cudaStream_t st, LaunchCounter* lc, const double* z, const double* dold, double* dnew,
                             double* xs, double* u, int nt, int n1, int n2, const AxisSym& s2, double scale,
                             const TimeFactor& tf, double psi, const double* a_num, const double* a_den,
                             const double* b_num, const double* b_den, bool first, bool upd_x,
                             const int* guard = nullptr);

// Preconditioner passes (pow2 lengths).
cudaError_t launch_hartley_row(cudaStream_t st, LaunchCounter* lc, const double* in, double* out, int F,
                               int n, const double2* tw, const double* rdot, RedSlot red,
                               const int* guard = nullptr);
cudaError_t launch_hartley_col(cudaStream_t st, LaunchCounter* lc, double* data, int O, int n, int C,
                               const double2* tw, const int* guard = nullptr);
cudaError_t launch_t_filter(cudaStream_t st, LaunchCounter* lc, double* data, const PcTables& pt,
                            const int* guard = nullptr);

// PCG control of one speculative iteration (1 thread): out[0] = pq,
// out[1] = |r|^2 (copied for the host); raises *pause when the host must act
// (pq <= 0 / non-finite, non-finite residual, or |r| <= tol |b|).
cudaError_t launch_pcg_control(cudaStream_t st, LaunchCounter* lc, const double* pq, const double* rr,
                               double tol_nb2, double* out, int* pause, const int* guard, double seq);
// Control step of the graph-driven PCG iterations (a CUDA graph whose WHILE
// node repeats a two-iteration body): ctl[1] counts iterations, ctl[2] is
// max_inner, *tol_nb2 the stop threshold (tol |b|)^2 of this solve.  Writes
// (pq, |r|^2, stop) of every iteration into out[4 (it & 1) ..]; when it stops
// (breakdown, |r| small, or the cap) it raises the pause flag, clears the
// WHILE condition and reports (pq, |r|^2, stop, it) in out[8..11], it last.
cudaError_t launch_pcg_control_graph(cudaStream_t st, LaunchCounter* lc, const double* pq, const double* rr,
                                     const double* tol_nb2, double* out, int* pause, int* ctl,
                                     cudaGraphConditionalHandle cond);
// PDL launch attributes off while this thread captures a graph body
void pdl_suspend(bool on);
// ctl[1] = it0 - 1, ctl[2] = max_inner, *tol_slot = tol_nb2 (stream ordered)
cudaError_t launch_pcg_graph_prep(cudaStream_t st, LaunchCounter* lc, int* ctl, int it0m1, int max_inner,
                                  double* tol_slot, double tol_nb2);

// ------------------------------------------------------------- elementwise
cudaError_t launch_copy(cudaStream_t st, LaunchCounter* lc, double* dst, const double* src, size_t N);
cudaError_t launch_fill(cudaStream_t st, LaunchCounter* lc, double* dst, double v, size_t N);
// Dense Hartley transform along one axis of length n (stride C, O outer
// blocks) with the cas table cas[m] = cos(2 pi m/n) + sin(2 pi m/n); and the
// 1/(N lambda_S) scaling of the 3-level preconditioner (any level sizes).
cudaError_t launch_cas_axis(cudaStream_t st, LaunchCounter* lc, const double* in, double* out, long O, int n,
                            long C, const double* cas);
cudaError_t launch_lams_scale(cudaStream_t st, LaunchCounter* lc, double* h, const PcTables& pt);
// *flag = 1 when some element of x is not zero (flag is not cleared)
cudaError_t launch_any_nonzero(cudaStream_t st, LaunchCounter* lc, const double* x, size_t N, int* flag);
// sum of squares (or dot when b != null) -> red.result[0]
// |a|^2, |b|^2 -> red.result[0..1] (one pass; partials need 2 x grid)
cudaError_t launch_norms2(cudaStream_t st, LaunchCounter* lc, const double* a, const double* b, size_t N,
                          RedSlot red);
cudaError_t launch_dot(cudaStream_t st, LaunchCounter* lc, const double* a, const double* b, size_t N,
                       RedSlot red);
// x += alpha p (alpha = num/den, optional), p = z + beta p (beta = bnum/bden)
cudaError_t launch_cg_update(cudaStream_t st, LaunchCounter* lc, double* x, double* p, const double* z,
                             size_t N, const double* a_num, const double* a_den, const double* b_num,
                             const double* b_den, bool update_x);
// x += alpha p only
cudaError_t launch_axpy_dev(cudaStream_t st, LaunchCounter* lc, double* x, const double* p, size_t N,
                            const double* a_num, const double* a_den, const int* guard = nullptr);
// r = b - q, reduce |r|^2
cudaError_t launch_residual(cudaStream_t st, LaunchCounter* lc, double* r, const double* b,
                            const double* q, size_t N, RedSlot red);
// out = a1[k] x (S with B == 0 part), used by the generic apply_S path
cudaError_t launch_scale_by_slice(cudaStream_t st, LaunchCounter* lc, double* out, const double* x,
                                  const double* coef, size_t slice, size_t N);

// ADMM elementwise stages (admm.cpp:100-119, 171-233) -- see fdg_kernels.cu.
struct AdmmScalars {
  double rho, delta, psi;
  double y_lo, y_hi, v_lo, v_hi;
};
cudaError_t launch_rhs_pre(cudaStream_t st, LaunchCounter* lc, const AdmmScalars& a, const double* p,
                           const double* w_v, const double* z_v, const double* a2inv,
                           const double* m2, double* r_cache, double* tmp, size_t slice, size_t N);
cudaError_t launch_rhs_post(cudaStream_t st, LaunchCounter* lc, const AdmmScalars& a, double* rhs,
                            const double* ybar, const double* w_y, const double* z_y,
                            const double* diag_j, size_t slice, size_t N);
// Fused recover_vp + z_update + dual_update + check_termination maxima + finiteness.
// red.result = {r_eq, r_y, r_v, nonfinite_flag}
cudaError_t launch_admm_update(cudaStream_t st, LaunchCounter* lc, const AdmmScalars& a, const double* y,
                               double* v, double* z_y, double* z_v, double* p, double* w_y,
                               double* w_v, const double* By, const double* r_cache,
                               const double* a2inv, const double* m2, size_t slice, size_t N,
                               RedSlot red);
// dual infeasibility maxima {s1, s2}
cudaError_t launch_dual_inf(cudaStream_t st, LaunchCounter* lc, const double* y, const double* ybar,
                            const double* btp, const double* w_y, const double* v, const double* p,
                            const double* w_v, const double* diag_j, const double* diag_j2,
                            size_t slice, size_t N, RedSlot red);
// objective {sum J (y - ybar)^2, sum J2 v^2}
cudaError_t launch_objective(cudaStream_t st, LaunchCounter* lc, const double* y, const double* ybar,
                             const double* v, const double* diag_j, const double* diag_j2,
                             size_t slice, size_t N, RedSlot red);

// Bluestein stages of the 2-level spatial preconditioner (fdg_kernels.cu).
// F = nt * n1 real rows; row-pair buffers are [F rounded up to even][n2],
// column-pair buffers [nt][n1][P2] with P2 = n2 rounded up to even.
// 1023-point prime-factor Hartley passes of the 2-level preconditioner
// (fdg_pfa.cu): rows out = scale * H2 in; columns in place H1 / lambda / H1.
bool pfa_supported(int n);
cudaError_t launch_pfa_hrow(cudaStream_t st, LaunchCounter* lc, const double* in, double* out, long F,
                            double scale);
cudaError_t launch_pfa_hcol(cudaStream_t st, LaunchCounter* lc, double* data, int nt, int C, const double* lam1,
                            const double* lam2);
cudaError_t launch_bs_pre_rows(cudaStream_t st, LaunchCounter* lc, const double* in, double* out, long F, int n2,
                               const double2* c2);
cudaError_t launch_bs_rows_to_cols(cudaStream_t st, LaunchCounter* lc, const double* v, double* u, long F, int n1,
                                   int n2, int P2, const double2* c2, const double2* c1);
cudaError_t launch_bs_cols_filter(cudaStream_t st, LaunchCounter* lc, const double* v, double* u, int nt, int n1,
                                  int n2, int P2, const double2* c1, const double* lam1, const double* lam2);
cudaError_t launch_bs_cols_to_rows(cudaStream_t st, LaunchCounter* lc, const double* v, double* u, long F, int n1,
                                   int n2, int P2, const double2* c1, const double2* c2);
cudaError_t launch_bs_post_rows(cudaStream_t st, LaunchCounter* lc, const double* v, double* z, long F, int n2,
                                const double2* c2, double scale);

// Grid of the reduction-bearing kernels (to size partial buffers).
size_t max_partials_needed(int nt, int n1, int n2);

}  // namespace fdg
