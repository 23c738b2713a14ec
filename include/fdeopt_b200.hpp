// include/fdeopt_b200.hpp — header-only C++ façade over include/fdg.h that
// keeps the reference's API (namespace fdeopt, /root/reference/proj/include/
// fdeopt/{toeplitz,circulant,admm}.hpp) so a caller can switch by changing the
// namespace and linking libfdg.so:
//
//   fdeopt::ConstraintOperator      -> fdeopt::b200::ConstraintOperator
//   fdeopt::assemble_precond        -> fdeopt::b200::assemble_precond
//   fdeopt::AdmmDriver / solve      -> fdeopt::b200::AdmmDriver / solve
//
// Differences, all additive: shapes may be (n_t, n_x1, n_x2) instead of n^3;
// the desired state and a fixed Krylov tolerance can be injected; device-
// pointer overloads exist next to the std::span host overloads.  Errors are
// the reference's: std::invalid_argument for parameters/dimensions and
// std::runtime_error (same message text) for numerical breakdowns.
#pragma once

#include <cmath>
#include <cstddef>
#include <limits>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "fdg.h"

namespace fdeopt::b200 {

inline void check(fdg_status s) {
  if (s == FDG_OK) return;
  const std::string msg = fdg_last_error();
  if (s == FDG_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

/// toeplitz.hpp:14-19
struct ToeplitzSpec1D {
  std::vector<double> col, row;
  int size() const { return static_cast<int>(col.size()); }
};

inline std::vector<double> frac_coeffs(double order, int count) {
  std::vector<double> g(count > 0 ? count : 0);
  check(fdg_frac_coeffs(order, count, g.data()));
  return g;
}

inline ToeplitzSpec1D build_riesz(double beta, int n, double h) {
  ToeplitzSpec1D s{std::vector<double>(n > 0 ? n : 0), std::vector<double>(n > 0 ? n : 0)};
  check(fdg_build_riesz(beta, n, h, s.col.data(), s.row.data()));
  return s;
}

inline ToeplitzSpec1D build_caputo(double alpha, int n, double h) {
  ToeplitzSpec1D s{std::vector<double>(n > 0 ? n : 0), std::vector<double>(n > 0 ? n : 0)};
  check(fdg_build_caputo(alpha, n, h, s.col.data(), s.row.data()));
  return s;
}

/// Implicit Euler = GL alpha = 1 bidiagonal factor.
inline ToeplitzSpec1D implicit_euler(int nt, double h_t) {
  ToeplitzSpec1D s{std::vector<double>(nt, 0.0), std::vector<double>(nt, 0.0)};
  s.col[0] = 1.0 / h_t;
  if (nt > 1) s.col[1] = -1.0 / h_t;
  s.row[0] = s.col[0];
  return s;
}

class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) {
    fdg_ctx c = nullptr;
    check(fdg_ctx_create(device, stream, &c));
    h_.reset(c);
  }
  fdg_ctx get() const { return h_.get(); }
  void synchronize() const { check(fdg_ctx_synchronize(h_.get())); }
  std::uint64_t launch_count() const { return fdg_ctx_launch_count(h_.get()); }

 private:
  struct D {
    void operator()(fdg_ctx c) const { fdg_ctx_destroy(c); }
  };
  std::unique_ptr<fdg_ctx_s, D> h_;
};

/// toeplitz.hpp:30-71
class ConstraintOperator {
 public:
  ConstraintOperator(const Context& ctx, const ToeplitzSpec1D& time, const ToeplitzSpec1D& x1,
                     const ToeplitzSpec1D& x2, double psi) {
    if (time.col.size() != time.row.size() || x1.col.size() != x1.row.size() ||
        x2.col.size() != x2.row.size())
      throw std::invalid_argument("ConstraintOperator: factor size mismatch");
    fdg_op o = nullptr;
    check(fdg_op_create(ctx.get(), time.size(), x1.size(), x2.size(), time.col.data(), time.row.data(),
                        x1.col.data(), x1.row.data(), x2.col.data(), x2.row.data(), psi, &o));
    h_.reset(o);
  }
  /// The reference's explicit-factor ctor (cube, toeplitz.cpp:87-101).
  ConstraintOperator(const Context& ctx, const ToeplitzSpec1D& caputo, const ToeplitzSpec1D& riesz1,
                     const ToeplitzSpec1D& riesz2, double psi, int n)
      : ConstraintOperator(ctx, caputo, riesz1, riesz2, psi) {
    if (caputo.size() != n || riesz1.size() != n || riesz2.size() != n)
      throw std::invalid_argument("ConstraintOperator: factor size mismatch");
  }

  /// toeplitz.hpp:55-56 (host spans; staged through the device)
  void apply(std::span<const double> x, std::span<double> out, bool adjoint = false) const {
    check(fdg_op_apply_host(h_.get(), x.data(), x.size(), out.data(), out.size(), adjoint ? 1 : 0));
  }
  std::vector<double> apply(std::span<const double> x, bool adjoint = false) const {
    std::vector<double> out(size());
    apply(x, out, adjoint);
    return out;
  }
  /// Device-resident overload (the hot path).
  void apply_device(const double* x_dev, double* out_dev, bool adjoint = false) const {
    check(fdg_op_apply(h_.get(), x_dev, out_dev, adjoint ? 1 : 0));
  }
  std::size_t size() const { return fdg_op_size(h_.get()); }
  double psi() const { return fdg_op_psi(h_.get()); }
  fdg_op get() const { return h_.get(); }

 private:
  struct D {
    void operator()(fdg_op o) const { fdg_op_destroy(o); }
  };
  std::unique_ptr<fdg_op_s, D> h_;
};

/// circulant.hpp:31-61
class CirculantPreconditioner {
 public:
  explicit CirculantPreconditioner(fdg_pc p, std::size_t n) : h_(p), n_(n) {}
  void solve(std::span<const double> r, std::span<double> z) const {
    check(fdg_pc_solve_host(h_.get(), r.data(), r.size(), z.data(), z.size()));
  }
  std::vector<double> solve(std::span<const double> r) const {
    std::vector<double> z(n_);
    solve(r, z);
    return z;
  }
  void solve_device(const double* r_dev, double* z_dev) const { check(fdg_pc_solve(h_.get(), r_dev, z_dev)); }
  std::vector<double> lam_s() const {
    std::vector<double> out(n_);
    check(fdg_pc_lam_s_host(h_.get(), out.data()));
    return out;
  }
  std::size_t size() const { return n_; }
  fdg_pc get() const { return h_.get(); }

 private:
  struct D {
    void operator()(fdg_pc p) const { fdg_pc_destroy(p); }
  };
  std::unique_ptr<fdg_pc_s, D> h_;
  std::size_t n_;
};

/// circulant.hpp:63-64
inline CirculantPreconditioner assemble_precond(const ConstraintOperator& op, double rho, double delta,
                                                double gamma) {
  fdg_pc p = nullptr;
  check(fdg_pc_assemble(op.get(), rho, delta, gamma, &p));
  return CirculantPreconditioner(p, op.size());
}

/// admm.hpp:14-26 (+ BASELINE's fixed Krylov tolerance)
struct AdmmConfig {
  double delta = 0.4;
  double rho = 1.618;
  double tol_primal = 1e-4;
  int max_outer = 500;
  double inner_tol_floor = 1e-4;
  double inner_tol_factor = 0.05;
  int max_inner = 400;
  bool warm_start = false;
  double fixed_krylov_tol = 0.0;  // > 0: fixed
};

inline constexpr double kUnbounded = std::numeric_limits<double>::infinity();

/// Bounds and gamma of ProblemSpec (problem.hpp:15-26).
struct Bounds {
  double gamma = 1e-4;
  double y_lo = -kUnbounded, y_hi = kUnbounded, u_lo = -kUnbounded, u_hi = kUnbounded;
};

/// admm.hpp:34-40
struct IterRecord {
  int iter;
  double r_eq, r_y, r_u;
  double dual_inf;
  int inner_iters;
  double inner_tol;
};

/// admm.hpp:86-90
struct PcgResult {
  int iterations = 0;
  bool converged = false;
  double rel_residual = 0.0;
};

enum class SolveStatus { converged, iteration_cap, failure };

/// admm.hpp:128-150
class AdmmDriver {
 public:
  AdmmDriver(const ConstraintOperator& op, const CirculantPreconditioner& pc, const Bounds& b,
             const AdmmConfig& cfg, std::span<const double> ybar = {})
      : cfg_(cfg), n_(op.size()) {
    const fdg_admm_desc d{b.gamma,        cfg.rho,         cfg.delta,        b.y_lo,
                          b.y_hi,         b.u_lo,          b.u_hi,           cfg.tol_primal,
                          cfg.max_outer,  cfg.max_inner,   cfg.inner_tol_floor, cfg.inner_tol_factor,
                          cfg.fixed_krylov_tol, cfg.warm_start ? 1 : 0};
    if (!ybar.empty() && ybar.size() != n_) throw std::invalid_argument("AdmmDriver: ybar size mismatch");
    fdg_admm a = nullptr;
    check(fdg_admm_create(op.get(), pc.get(), &d, ybar.empty() ? nullptr : ybar.data(), &a));
    h_.reset(a);
  }

  IterRecord step() {
    fdg_iter_record r{};
    check(fdg_admm_step(h_.get(), &r));
    return IterRecord{r.iter, r.r_eq, r.r_y, r.r_u, r.dual_inf, r.inner_iters, r.inner_tol};
  }
  bool converged() const { return fdg_admm_converged(h_.get()) != 0; }
  int consecutive_stagnations() const { return fdg_admm_stagnations(h_.get()); }

  std::vector<double> field(int f) const {
    std::vector<double> out(n_);
    check(fdg_admm_get(h_.get(), f, out.data()));
    return out;
  }
  std::vector<double> y() const { return field(FDG_F_Y); }
  std::vector<double> v() const { return field(FDG_F_V); }
  std::vector<double> p() const { return field(FDG_F_P); }

  /// pcg(apply_S, pc.solve, rhs, x, tol, max_inner) on this driver's work.
  PcgResult pcg(std::span<const double> rhs, std::vector<double>& x, double tol, int max_inner) {
    if (rhs.size() != n_) throw std::invalid_argument("pcg: dimension mismatch");
    if (x.size() != n_) x.assign(n_, 0.0);
    fdg_pcg_result r{};
    check(fdg_admm_pcg_host(h_.get(), rhs.data(), x.data(), tol, max_inner, &r));
    return PcgResult{r.iterations, r.converged != 0, r.rel_residual};
  }
  double dual_infeasibility() const {
    double d = 0.0;
    check(fdg_admm_dual_inf(h_.get(), &d));
    return d;
  }
  double objective() const {
    double d = 0.0;
    check(fdg_admm_objective(h_.get(), &d));
    return d;
  }
  const AdmmConfig& config() const { return cfg_; }
  std::size_t size() const { return n_; }

 private:
  struct D {
    void operator()(fdg_admm a) const { fdg_admm_destroy(a); }
  };
  std::unique_ptr<fdg_admm_s, D> h_;
  AdmmConfig cfg_;
  std::size_t n_;
};

struct SolveResult {
  int iterations = 0;
  double pcg_avg = 0.0;
  double dual_inf = 0.0;
  double objective = 0.0;
  SolveStatus status = SolveStatus::failure;
  std::vector<IterRecord> history;
};

/// admm.cpp:279-324 outer loop (3 consecutive PCG caps -> runtime_error).
inline SolveResult solve(AdmmDriver& driver) {
  SolveResult res;
  long total_inner = 0;
  for (int j = 0; j < driver.config().max_outer; ++j) {
    const IterRecord rec = driver.step();
    total_inner += rec.inner_iters;
    res.history.push_back(rec);
    if (driver.consecutive_stagnations() >= 3)
      throw std::runtime_error("admm: PCG hit max_inner in 3 consecutive outer iterations");
    if (driver.converged()) break;
  }
  res.iterations = static_cast<int>(res.history.size());
  res.pcg_avg = res.iterations ? static_cast<double>(total_inner) / res.iterations : 0.0;
  res.status = driver.converged() ? SolveStatus::converged : SolveStatus::iteration_cap;
  res.dual_inf = driver.dual_infeasibility();
  res.objective = driver.objective();
  return res;
}

}  // namespace fdeopt::b200
