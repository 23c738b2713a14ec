// oracle/ref_adapter.cpp — TEST INFRASTRUCTURE (checker + CPU baseline only).
//
// A C ABI (for ctypes) over the UNCHANGED reference sources
// /root/reference/proj/src/{fft,problem,toeplitz,circulant,admm}.cpp, compiled
// with the FFTW3 shim in oracle/shim.  Nothing here re-implements reference
// arithmetic: every number comes out of the reference's own public functions.
// The only driver-level change is the one SURVEY.md Appendix A asks for: the
// ADMM step is re-sequenced from the public free functions in exactly the order
// of AdmmDriver::step (admm.cpp:245-277) so that (a) the desired state ybar can
// be injected through AdmmWork::ybar (admm.hpp:66) and (b) the Krylov
// tolerance can be fixed (BASELINE) instead of the dynamic rule
// (admm.cpp:216-217).  With ybar=NULL and fixed_tol<=0 it is AdmmDriver::step.
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "fdeopt/admm.hpp"
#include "fdeopt/circulant.hpp"
#include "fdeopt/problem.hpp"
#include "fdeopt/toeplitz.hpp"
#include "minifft.h"

using namespace fdeopt;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -3;
  }
}

std::vector<double> vec(const double* p, std::size_t n) { return std::vector<double>(p, p + n); }

void put_complex(const std::vector<fft::Complex>& v, double* out) {
  for (std::size_t i = 0; i < v.size(); ++i) {
    out[2 * i] = v[i].real();
    out[2 * i + 1] = v[i].imag();
  }
}

struct OpHandle {
  std::unique_ptr<ConstraintOperator> op;
  ConstraintOperator::Workspace ws;
};

struct PcHandle {
  std::unique_ptr<CirculantPreconditioner> pc;
  CirculantPreconditioner::Workspace ws;
};

struct AdmmHandle {
  OpHandle* op;
  PcHandle* pc;
  AdmmWork work;
  AdmmState state;
  std::vector<double> By;
  double inner_tol;
  double fixed_tol;  // > 0: BASELINE fixed Krylov tolerance
  bool converged = false;
  int stagnations = 0;
  double pcg_seconds_total = 0.0;
  long inner_total = 0;
};

enum Field { F_Y = 0, F_V, F_ZY, F_ZV, F_P, F_WY, F_WV, F_YBAR, F_DIAGJ, F_DIAGJ2, F_M2, F_A2INV, F_BY };

std::vector<double>* field_ptr(AdmmHandle* h, int f) {
  switch (f) {
    case F_Y: return &h->state.y;
    case F_V: return &h->state.v;
    case F_ZY: return &h->state.z_y;
    case F_ZV: return &h->state.z_v;
    case F_P: return &h->state.p;
    case F_WY: return &h->state.w_y;
    case F_WV: return &h->state.w_v;
    case F_YBAR: return &h->work.ybar;
    case F_DIAGJ: return &h->work.diag_j;
    case F_DIAGJ2: return &h->work.diag_j2;
    case F_M2: return &h->work.m2;
    case F_A2INV: return &h->work.a2_inv;
    case F_BY: return &h->By;
    default: throw std::invalid_argument("ref_admm: unknown field");
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int t) { mf_set_threads(t); }

// problem.cpp:35-45
int ref_frac_coeffs(double order, int count, double* out) {
  return guard([&] {
    const auto g = frac_coeffs(order, count);
    std::memcpy(out, g.data(), sizeof(double) * g.size());
  });
}

// problem.cpp:26-33 (validates the spec, so alpha must lie in (0,1))
int ref_scaling(double alpha, double beta1, double beta2, int n, double* out4) {
  return guard([&] {
    ProblemSpec spec;
    spec.alpha = alpha;
    spec.beta1 = beta1;
    spec.beta2 = beta2;
    spec.n = n;
    const auto s = scaling(spec, Grid(n));
    out4[0] = s.psi;
    out4[1] = s.nu1;
    out4[2] = s.nu2;
    out4[3] = s.nu3;
  });
}

// problem.cpp:47-58
int ref_desired_state(int n, double* out) {
  return guard([&] {
    const auto v = desired_state(Grid(n));
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  });
}

// toeplitz.cpp:10-21
int ref_build_caputo(double alpha, int n, double h_t, double* col, double* row) {
  return guard([&] {
    const auto s = build_caputo(alpha, n, h_t);
    std::memcpy(col, s.col.data(), sizeof(double) * n);
    std::memcpy(row, s.row.data(), sizeof(double) * n);
  });
}

// toeplitz.cpp:23-42
int ref_build_riesz(double beta, int n, double h_x, double* col, double* row) {
  return guard([&] {
    const auto s = build_riesz(beta, n, h_x);
    std::memcpy(col, s.col.data(), sizeof(double) * n);
    std::memcpy(row, s.row.data(), sizeof(double) * n);
  });
}

// toeplitz.cpp:62-79
int ref_toeplitz_matvec(int n, const double* col, const double* row, const double* x, double* out,
                        int transpose) {
  return guard([&] {
    ToeplitzSpec1D s{vec(col, n), vec(row, n)};
    const auto y = toeplitz_matvec(s, std::span<const double>(x, n), transpose != 0);
    std::memcpy(out, y.data(), sizeof(double) * n);
  });
}

// toeplitz.cpp:46-58 -> n+1 complex bins (interleaved re/im)
int ref_embed_symbol(int n, const double* col, const double* row, int transpose, double* sym) {
  return guard([&] {
    ToeplitzSpec1D s{vec(col, n), vec(row, n)};
    put_complex(detail::embed_symbol(s, transpose != 0), sym);
  });
}

// circulant.cpp:10-20
int ref_tchan(int n, const double* col, const double* row, double* first_col, double* eigs) {
  return guard([&] {
    ToeplitzSpec1D s{vec(col, n), vec(row, n)};
    const auto c = tchan(s);
    std::memcpy(first_col, c.first_col.data(), sizeof(double) * n);
    put_complex(c.eigs, eigs);
  });
}

// circulant.cpp:22-26
int ref_circulant_eigs(int n, const double* first_col, double* eigs) {
  return guard([&] { put_complex(circulant_eigs(std::span<const double>(first_col, n)), eigs); });
}

// fft.cpp:111-130
int ref_dft(int n, const double* in, double* out, int inverse) {
  return guard([&] {
    std::vector<fft::Complex> x(n);
    for (int i = 0; i < n; ++i) x[i] = {in[2 * i], in[2 * i + 1]};
    put_complex(fft::dft(x, inverse != 0), out);
  });
}

// ConstraintOperator explicit-factor ctor, toeplitz.cpp:87-101
void* ref_op_create(int n, const double* tcol, const double* trow, const double* c1,
                    const double* r1, const double* c2, const double* r2, double psi) {
  OpHandle* h = nullptr;
  const int rc = guard([&] {
    auto op = std::make_unique<ConstraintOperator>(ToeplitzSpec1D{vec(tcol, n), vec(trow, n)},
                                                   ToeplitzSpec1D{vec(c1, n), vec(r1, n)},
                                                   ToeplitzSpec1D{vec(c2, n), vec(r2, n)}, psi, n);
    h = new OpHandle{std::move(op), {}};
    h->ws = h->op->make_workspace();
  });
  return rc == 0 ? h : nullptr;
}

// ConstraintOperator(spec, grid), toeplitz.cpp:81-85
void* ref_op_create_spec(double alpha, double beta1, double beta2, int n) {
  OpHandle* h = nullptr;
  const int rc = guard([&] {
    ProblemSpec spec;
    spec.alpha = alpha;
    spec.beta1 = beta1;
    spec.beta2 = beta2;
    spec.n = n;
    auto op = std::make_unique<ConstraintOperator>(spec, Grid(n));
    h = new OpHandle{std::move(op), {}};
    h->ws = h->op->make_workspace();
  });
  return rc == 0 ? h : nullptr;
}

// ConstraintOperator::zero, toeplitz.cpp:103-108
void* ref_op_create_zero(int n) {
  OpHandle* h = nullptr;
  const int rc = guard([&] {
    auto op = std::make_unique<ConstraintOperator>(ConstraintOperator::zero(n));
    h = new OpHandle{std::move(op), {}};
    h->ws = h->op->make_workspace();
  });
  return rc == 0 ? h : nullptr;
}

void ref_op_destroy(void* h) { delete static_cast<OpHandle*>(h); }

double ref_op_psi(void* h) { return static_cast<OpHandle*>(h)->op->psi(); }

// toeplitz.cpp:174-182
int ref_op_apply(void* vh, const double* x, double* out, long n_x, long n_out, int adjoint) {
  auto* h = static_cast<OpHandle*>(vh);
  return guard([&] {
    h->op->apply(std::span<const double>(x, n_x), std::span<double>(out, n_out), h->ws,
                 adjoint != 0);
  });
}

// circulant.cpp:76-90
void* ref_pc_assemble(void* vop, double rho, double delta, double gamma) {
  PcHandle* h = nullptr;
  const int rc = guard([&] {
    auto* op = static_cast<OpHandle*>(vop);
    auto pc = std::make_unique<CirculantPreconditioner>(assemble_precond(*op->op, rho, delta, gamma));
    h = new PcHandle{std::move(pc), {}};
    h->ws = h->pc->make_workspace();
  });
  return rc == 0 ? h : nullptr;
}

// circulant.cpp:28-41
void* ref_pc_create(const double* lam_b, int n, double rho, double delta, double gamma,
                    double psi) {
  PcHandle* h = nullptr;
  const int rc = guard([&] {
    const std::size_t N = static_cast<std::size_t>(n) * n * n;
    std::vector<fft::Complex> lb(N);
    for (std::size_t i = 0; i < N; ++i) lb[i] = {lam_b[2 * i], lam_b[2 * i + 1]};
    auto pc = std::make_unique<CirculantPreconditioner>(std::move(lb), rho, delta, gamma, psi, n);
    h = new PcHandle{std::move(pc), {}};
    h->ws = h->pc->make_workspace();
  });
  return rc == 0 ? h : nullptr;
}

void ref_pc_destroy(void* h) { delete static_cast<PcHandle*>(h); }

// circulant.cpp:49-67
int ref_pc_solve(void* vh, const double* r, double* z, long n_r, long n_z) {
  auto* h = static_cast<PcHandle*>(vh);
  return guard([&] {
    h->pc->solve(std::span<const double>(r, n_r), std::span<double>(z, n_z), h->ws);
  });
}

int ref_pc_lam_s(void* vh, double* out) {
  auto* h = static_cast<PcHandle*>(vh);
  return guard([&] {
    std::memcpy(out, h->pc->lam_s().data(), sizeof(double) * h->pc->lam_s().size());
  });
}

int ref_pc_lam_b(void* vh, double* out) {
  auto* h = static_cast<PcHandle*>(vh);
  return guard([&] { put_complex(h->pc->lam_b(), out); });
}

// ------------------------------------------------------------------ ADMM

// make_admm_work (admm.cpp:52-79) needs spec.validate(); alpha/betas are only
// validated, never used there, so the BASELINE adapter passes placeholders.
void* ref_admm_create(void* vop, void* vpc, double gamma, double rho, double delta, double y_lo,
                      double y_hi, double u_lo, double u_hi, double tol_primal, int max_outer,
                      int max_inner, double inner_tol_floor, double inner_tol_factor,
                      double fixed_tol, int warm_start, const double* ybar) {
  AdmmHandle* h = nullptr;
  const int rc = guard([&] {
    auto* op = static_cast<OpHandle*>(vop);
    ProblemSpec spec;
    spec.alpha = 0.5;
    spec.beta1 = 1.5;
    spec.beta2 = 1.5;
    spec.gamma = gamma;
    spec.n = op->op->n();
    spec.y_lo = y_lo;
    spec.y_hi = y_hi;
    spec.u_lo = u_lo;
    spec.u_hi = u_hi;
    AdmmConfig cfg;
    cfg.rho = rho;
    cfg.delta = delta;
    cfg.tol_primal = tol_primal;
    cfg.max_outer = max_outer;
    cfg.max_inner = max_inner;
    cfg.inner_tol_floor = inner_tol_floor;
    cfg.inner_tol_factor = inner_tol_factor;
    cfg.warm_start = warm_start != 0;
    h = new AdmmHandle{op, static_cast<PcHandle*>(vpc), make_admm_work(spec, cfg, *op->op),
                       zero_state(op->op->size()), {}, 0.0, fixed_tol};
    h->By.assign(h->work.size(), 0.0);
    h->inner_tol = cfg.inner_tol_factor * cfg.inner_tol_floor;  // admm.cpp:245
    if (ybar) h->work.ybar = vec(ybar, h->work.size());
  });
  return rc == 0 ? h : nullptr;
}

void ref_admm_destroy(void* h) { delete static_cast<AdmmHandle*>(h); }

long ref_admm_size(void* vh) { return static_cast<long>(static_cast<AdmmHandle*>(vh)->work.size()); }
double ref_admm_psi(void* vh) { return static_cast<AdmmHandle*>(vh)->work.psi; }

int ref_admm_get(void* vh, int field, double* out) {
  auto* h = static_cast<AdmmHandle*>(vh);
  return guard([&] {
    const auto* v = field_ptr(h, field);
    std::memcpy(out, v->data(), sizeof(double) * v->size());
  });
}

int ref_admm_set(void* vh, int field, const double* in) {
  auto* h = static_cast<AdmmHandle*>(vh);
  return guard([&] {
    auto* v = field_ptr(h, field);
    std::memcpy(v->data(), in, sizeof(double) * v->size());
  });
}

// admm.cpp:87-98
int ref_admm_apply_S(void* vh, const double* x, double* out) {
  auto* h = static_cast<AdmmHandle*>(vh);
  return guard([&] {
    const std::size_t N = h->work.size();
    apply_S(h->work, std::span<const double>(x, N), std::span<double>(out, N), h->op->ws);
  });
}

// admm.cpp:100-119
int ref_admm_build_rhs(void* vh, double* rhs, double* r_cache) {
  auto* h = static_cast<AdmmHandle*>(vh);
  return guard([&] {
    std::vector<double> rv;
    const auto r = build_rhs(h->work, h->state, rv, h->op->ws);
    std::memcpy(rhs, rv.data(), sizeof(double) * rv.size());
    if (r_cache) std::memcpy(r_cache, r.data(), sizeof(double) * r.size());
  });
}

// admm.cpp:121-169 on the ADMM normal equations (apply_S + pc.solve).
// result: {iterations, converged, rel_residual, seconds}
int ref_admm_pcg(void* vh, const double* rhs, double* x, double tol, int max_inner,
                 double* result) {
  auto* h = static_cast<AdmmHandle*>(vh);
  return guard([&] {
    const std::size_t N = h->work.size();
    LinearFn apply = [&](std::span<const double> a, std::span<double> b) {
      apply_S(h->work, a, b, h->op->ws);
    };
    LinearFn precond = [&](std::span<const double> a, std::span<double> b) {
      h->pc->pc->solve(a, b, h->pc->ws);
    };
    std::vector<double> xv = vec(x, N);
    const auto t0 = std::chrono::steady_clock::now();
    const PcgResult res = pcg(apply, precond, std::span<const double>(rhs, N), xv, tol, max_inner);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::memcpy(x, xv.data(), sizeof(double) * N);
    result[0] = res.iterations;
    result[1] = res.converged ? 1.0 : 0.0;
    result[2] = res.rel_residual;
    result[3] = secs;
  });
}

// pcg's start (admm.cpp:125-141, x == 0 path): r = rhs, z = M r, p = z, rz = r.z
int ref_admm_krylov_init(void* vh, const double* rhs, double* r, double* z, double* p, double* rz) {
  auto* h = static_cast<AdmmHandle*>(vh);
  return guard([&] {
    const std::size_t N = h->work.size();
    std::memcpy(r, rhs, sizeof(double) * N);
    h->pc->pc->solve(std::span<const double>(r, N), std::span<double>(z, N), h->pc->ws);
    std::memcpy(p, z, sizeof(double) * N);
    double s = 0.0;
    for (std::size_t i = 0; i < N; ++i) s += r[i] * z[i];
    *rz = s;
  });
}

// Exactly one iteration of pcg's loop body (admm.cpp:142-163) with the
// reference's apply_S and CirculantPreconditioner::solve: the bounded unit of
// the CPU baseline.  out = {pq, |r|, rz_next}; *rz is updated.
int ref_admm_krylov_iteration(void* vh, double* x, double* r, double* z, double* p, double* q,
                              double* rz, double* out) {
  auto* h = static_cast<AdmmHandle*>(vh);
  return guard([&] {
    const std::size_t N = h->work.size();
    apply_S(h->work, std::span<const double>(p, N), std::span<double>(q, N), h->op->ws);
    double pq = 0.0;
    for (std::size_t i = 0; i < N; ++i) pq += p[i] * q[i];
    if (!std::isfinite(pq) || pq <= 0.0)
      throw std::runtime_error("pcg: operator lost positive definiteness");
    const double a = *rz / pq;
    for (std::size_t i = 0; i < N; ++i) {
      x[i] += a * p[i];
      r[i] -= a * q[i];
    }
    double rr = 0.0;
    for (std::size_t i = 0; i < N; ++i) rr += r[i] * r[i];
    h->pc->pc->solve(std::span<const double>(r, N), std::span<double>(z, N), h->pc->ws);
    double rzn = 0.0;
    for (std::size_t i = 0; i < N; ++i) rzn += r[i] * z[i];
    const double beta = rzn / *rz;
    *rz = rzn;
    for (std::size_t i = 0; i < N; ++i) p[i] = z[i] + beta * p[i];
    out[0] = pq;
    out[1] = std::sqrt(rr);
    out[2] = rzn;
  });
}

// AdmmDriver::step, admm.cpp:245-277, re-sequenced from the public functions.
// rec: {iter, r_eq, r_y, r_u, dual_inf, inner_iters, inner_tol, converged,
//       pcg_seconds, step_seconds, pcg_rel_residual, stagnations}
int ref_admm_step(void* vh, double* rec) {
  auto* h = static_cast<AdmmHandle*>(vh);
  return guard([&] {
    const auto t_step = std::chrono::steady_clock::now();
    const AdmmWork& work = h->work;
    auto& st = h->state;
    std::vector<double> rhs;
    const std::vector<double> r_cache = build_rhs(work, st, rhs, h->op->ws);
    LinearFn apply = [&](std::span<const double> x, std::span<double> out) {
      apply_S(work, x, out, h->op->ws);
    };
    LinearFn precond = [&](std::span<const double> r, std::span<double> z) {
      h->pc->pc->solve(r, z, h->pc->ws);
    };
    if (!work.cfg.warm_start) st.y.assign(work.size(), 0.0);
    const double tol = h->fixed_tol > 0.0 ? h->fixed_tol : h->inner_tol;
    const auto t0 = std::chrono::steady_clock::now();
    const PcgResult inner = pcg(apply, precond, rhs, st.y, tol, work.cfg.max_inner);
    const double pcg_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    h->stagnations = inner.converged ? 0 : h->stagnations + 1;
    h->op->op->apply(st.y, h->By, h->op->ws, false);
    std::vector<double> p_tilde;
    recover_vp(work, st, h->By, r_cache, st.v, p_tilde);
    z_update(work, st);
    dual_update(work, st, h->By);
    ++st.iteration;
    for (const auto* v : {&st.y, &st.v, &st.p})
      for (double d : *v)
        if (!std::isfinite(d))
          throw std::runtime_error("admm: non-finite iterate at outer iteration " +
                                   std::to_string(st.iteration));
    const Termination t = check_termination(work, st, h->By);
    h->converged = t.converged;
    h->inner_tol = t.inner_tol;
    const double dinf = dual_infeasibility(work, st, h->op->ws);
    h->pcg_seconds_total += pcg_s;
    h->inner_total += inner.iterations;
    rec[0] = st.iteration;
    rec[1] = t.r_eq;
    rec[2] = t.r_y;
    rec[3] = t.r_u;
    rec[4] = dinf;
    rec[5] = inner.iterations;
    rec[6] = t.inner_tol;
    rec[7] = t.converged ? 1.0 : 0.0;
    rec[8] = pcg_s;
    rec[9] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_step).count();
    rec[10] = inner.rel_residual;
    rec[11] = h->stagnations;
  });
}

// admm.cpp:221-233
int ref_admm_dual_inf(void* vh, double* out) {
  auto* h = static_cast<AdmmHandle*>(vh);
  return guard([&] { *out = dual_infeasibility(h->work, h->state, h->op->ws); });
}

// SURVEY.md §8 a19 (absent in the reference): Phi = 1/2 (y-ybar)^T J (y-ybar)
// + 1/2 v^T J2 v, evaluated on the reference's own state vectors.
int ref_admm_objective(void* vh, double* out) {
  auto* h = static_cast<AdmmHandle*>(vh);
  return guard([&] {
    const auto& w = h->work;
    const auto& s = h->state;
    double a = 0.0, b = 0.0;
    for (std::size_t i = 0; i < w.size(); ++i) {
      const double d = s.y[i] - w.ybar[i];
      a += w.diag_j[i] * d * d;
      b += w.diag_j2[i] * s.v[i] * s.v[i];
    }
    *out = 0.5 * a + 0.5 * b;
  });
}

// fdeopt::solve (admm.cpp:279-324), unchanged, for the reference's own
// experiment.  summary: {status(0 conv,1 cap), iterations, pcg_avg, misfit,
// dual_inf, wall_seconds}; history rows of 7: iter,r_eq,r_y,r_u,dual_inf,
// inner_iters,inner_tol.  Returns history length in *n_hist (<= hist_cap).
int ref_solve(double alpha, double beta1, double beta2, double gamma, int n, double y_lo,
              double y_hi, double u_lo, double u_hi, double delta, double rho, double tol_primal,
              int max_outer, int max_inner, int warm_start, double* summary, double* history,
              int hist_cap, int* n_hist, double* y_out, double* u_out) {
  return guard([&] {
    ProblemSpec spec;
    spec.alpha = alpha;
    spec.beta1 = beta1;
    spec.beta2 = beta2;
    spec.gamma = gamma;
    spec.n = n;
    spec.y_lo = y_lo;
    spec.y_hi = y_hi;
    spec.u_lo = u_lo;
    spec.u_hi = u_hi;
    AdmmConfig cfg;
    cfg.delta = delta;
    cfg.rho = rho;
    cfg.tol_primal = tol_primal;
    cfg.max_outer = max_outer;
    cfg.max_inner = max_inner;
    cfg.warm_start = warm_start != 0;
    const SolveResult r = solve(spec, cfg);
    summary[0] = r.status == SolveStatus::converged ? 0.0 : 1.0;
    summary[1] = r.iterations;
    summary[2] = r.pcg_avg;
    summary[3] = r.misfit;
    summary[4] = r.dual_inf;
    summary[5] = r.wall_seconds;
    int k = 0;
    for (const auto& rec : r.history) {
      if (k >= hist_cap) break;
      double* row = history + 7 * k;
      row[0] = rec.iter;
      row[1] = rec.r_eq;
      row[2] = rec.r_y;
      row[3] = rec.r_u;
      row[4] = rec.dual_inf;
      row[5] = rec.inner_iters;
      row[6] = rec.inner_tol;
      ++k;
    }
    *n_hist = k;
    if (y_out) std::memcpy(y_out, r.y.data(), sizeof(double) * r.y.size());
    if (u_out) std::memcpy(u_out, r.u.data(), sizeof(double) * r.u.size());
  });
}

// The reference tests' RNG: std::mt19937_64(seed) + std::normal_distribution
// (libstdc++), drawn in layout order (test_toeplitz.cpp:15-20).
int ref_randn(uint64_t seed, long count, double* out) {
  return guard([&] {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss;
    for (long i = 0; i < count; ++i) out[i] = gauss(rng);
  });
}

}  // extern "C"
