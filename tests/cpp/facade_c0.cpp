// A reference-style C++ caller of the B200 path through include/fdeopt_b200.hpp:
// builds the BASELINE C0 operator / preconditioner / driver the way a user of
// fdeopt would (explicit-factor ctor, assemble_precond, AdmmDriver::step),
// runs 5 ADMM steps and prints the per-step Krylov counts and residuals.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "fdeopt_b200.hpp"

int main() {
  using namespace fdeopt::b200;
  const int n = 8;
  const double ht = 1.0 / n, h = 1.0 / (n + 1);
  Context ctx(0);
  const auto time = implicit_euler(n, ht);
  const auto r = build_riesz(1.5, n, h);
  const double psi = std::min(ht, std::pow(h, 1.5));
  ConstraintOperator op(ctx, time, r, r, psi, n);
  auto pc = assemble_precond(op, 1.0, 1.0, 1e-4);
  // desired state: sin(pi x1) sin(pi x2) e^t + 0.01 N(0,1), seed 1
  std::vector<double> ybar(op.size());
  std::mt19937_64 rng(1);
  std::normal_distribution<double> gauss;
  const double pi = 3.14159265358979323846;
  for (int k = 0; k < n; ++k)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        ybar[(k * n + i) * n + j] =
            std::sin(pi * (i + 1) * h) * std::sin(pi * (j + 1) * h) * std::exp((k + 1) * ht);
  for (auto& v : ybar) v += 0.01 * gauss(rng);
  AdmmConfig cfg;
  cfg.delta = 1.0;
  cfg.rho = 1.0;
  cfg.tol_primal = 1e-6;
  cfg.fixed_krylov_tol = 1e-8;
  Bounds b;
  b.u_lo = -2.0;
  b.u_hi = 1.5;
  AdmmDriver drv(op, pc, b, cfg, ybar);
  for (int s = 0; s < 5; ++s) {
    const IterRecord rec = drv.step();
    std::printf("step %d inner %d r_eq %.17g r_u %.17g dual_inf %.17g\n", rec.iter, rec.inner_iters, rec.r_eq,
                rec.r_u, rec.dual_inf);
  }
  std::printf("objective %.17g\n", drv.objective());
  try {
    op.apply(std::vector<double>(3));
    std::printf("ERROR: size mismatch not detected\n");
    return 1;
  } catch (const std::invalid_argument&) {
    std::printf("size check ok\n");
  }
  return 0;
}
