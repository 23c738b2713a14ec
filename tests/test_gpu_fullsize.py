"""Parity at the BASELINE sizes the bench times.

* C2 (256^3) against the UNCHANGED reference (oracle/_ref, cube-capable):
  B, B^T, M^-1 and S on seeded N(0,1) vectors within 1e-11 (2-norm relative,
  SURVEY App. A.9), then the first two ADMM steps (build_rhs -> PCG ->
  recover / z / dual updates -> residuals -> dual_inf): Krylov count +-1 per
  step, r_eq, r_y, r_u, dual_inf within 1e-8 relative, y, v, p within 1e-8.
  These launch exactly the kernels bench.py times at C2 (k_rowc<512,*>,
  k_colc<512,2>, k_hartley_row/col<256>, k_t_filter<256>).
* C3 (128x512^2) and C4 (128x1024^2) with their real BASELINE parameters
  (orders, d_y, gamma, state box, target state) against the generalized C
  restatement (oracle/build, fibre-parallel): B, B^T, M^-1, S within 1e-11 and
  one PCG solve of the first ADMM sub-problem, Krylov count +-1 (k_rowq<1024>,
  k_colc<1024,2>, k_rowc<2048,*>, k_colc<2048,2>, k_t_filter<128>).

Reference: toeplitz.cpp:174-182, circulant.cpp:49-67, admm.cpp:87-98,
121-169, 245-277.  Host-side oracle runs use every host core (the reference's
loops stay serial; only its FFT batches / the port's fibre loops are split).
"""
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

OP_TOL = 1e-11
RES_TOL = 1e-8


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _close(got, exp, tol=RES_TOL):
    return abs(got - exp) <= tol * abs(exp) + 1e-300


def test_c2_fullsize_vs_reference(gpu_ctx, ref):
    from oracle import Shape, baseline_problem, synthetic_ybar
    from oracle.pyoracle import RefAdmm
    from paper_1907_13428_b200 import AdmmConfig, AdmmDriver, ConstraintOperator, assemble_precond
    ref.set_threads(_cores())
    s = Shape(256, 256, 256)
    n = s.nt
    c = baseline_problem("C2", s)
    yb = synthetic_ybar("sin", s)
    rop = ref.op(n, c["time"], c["r1"], c["r2"], c["psi"])
    rpc = rop.assemble_precond(1.0, 1.0, c["gamma"])
    radm = RefAdmm(ref, rop, rpc, c["gamma"], 1.0, 1.0, u_lo=c["u"][0], u_hi=c["u"][1],
                   tol_primal=1e-6, max_inner=400, fixed_tol=1e-8, ybar=yb)
    op = ConstraintOperator(c["time"], c["r1"], c["r2"], c["psi"], ctx=gpu_ctx)
    pc = assemble_precond(op, 1.0, 1.0, c["gamma"])
    cfg = AdmmConfig(delta=1.0, rho=1.0, tol_primal=1e-6, max_outer=100000, max_inner=400,
                     fixed_krylov_tol=1e-8)
    drv = AdmmDriver(op, pc, c["gamma"], cfg, u_lo=c["u"][0], u_hi=c["u"][1], ybar=yb)

    x = ref.randn(101, s.N)
    errs = {"B": rel(op.apply(x), rop.apply(x)), "BT": rel(op.apply(x, True), rop.apply(x, True)),
            "Minv": rel(pc.solve(x), rpc.solve(x)), "S": rel(drv.apply_S(x), radm.apply_S(x))}
    print("C2 256^3 vs reference:", {k: f"{v:.2e}" for k, v in errs.items()})
    assert max(errs.values()) < OP_TOL, errs

    for step in range(2):
        g, r = drv.step(), radm.step()
        print(f"step {step + 1}: krylov gpu {g.inner_iters} ref {r['inner_iters']}; "
              f"r_eq {g.r_eq:.6e}/{r['r_eq']:.6e} r_u {g.r_u:.6e}/{r['r_u']:.6e} "
              f"dual_inf {g.dual_inf:.6e}/{r['dual_inf']:.6e}")
        assert abs(g.inner_iters - r["inner_iters"]) <= 1
        for k in ("r_eq", "r_y", "r_u", "dual_inf"):
            assert _close(getattr(g, k), r[k]), (step, k, getattr(g, k), r[k])
        for f in ("y", "v", "p"):
            e = rel(drv.get(f), radm.get(f))
            assert e < RES_TOL, (step, f, e)


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_fullsize_vs_port(gpu_ctx, port, name):
    from oracle import Shape, baseline_problem
    from oracle.pyoracle import PortAdmm
    from paper_1907_13428_b200 import AdmmConfig, AdmmDriver, ConstraintOperator, assemble_precond
    from paper_1907_13428_b200.workloads import synthetic_ybar
    port.set_threads(_cores())
    c = baseline_problem(name)
    shape = c["shape"].tuple()
    yb = synthetic_ybar(c["ybar"], shape)
    pop = port.op(shape, c["time"], c["r1"], c["r2"], c["psi"])
    ppc = pop.assemble_precond(1.0, 1.0, c["gamma"])
    padm = PortAdmm(port, pop, ppc, c["gamma"], 1.0, 1.0, y_lo=c["y"][0], y_hi=c["y"][1],
                    u_lo=c["u"][0], u_hi=c["u"][1], tol_primal=1e-6, max_inner=400,
                    fixed_tol=1e-8, ybar=yb)
    op = ConstraintOperator(c["time"], c["r1"], c["r2"], c["psi"], shape=shape, ctx=gpu_ctx)
    pc = assemble_precond(op, 1.0, 1.0, c["gamma"])
    cfg = AdmmConfig(delta=1.0, rho=1.0, tol_primal=1e-6, max_outer=100000, max_inner=400,
                     fixed_krylov_tol=1e-8)
    drv = AdmmDriver(op, pc, c["gamma"], cfg, y_lo=c["y"][0], y_hi=c["y"][1], u_lo=c["u"][0],
                     u_hi=c["u"][1], ybar=yb)

    x = np.random.default_rng(7).standard_normal(pop.size)
    errs = {"B": rel(op.apply(x), pop.apply(x)), "BT": rel(op.apply(x, True), pop.apply(x, True)),
            "Minv": rel(pc.solve(x), ppc.solve(x)), "S": rel(drv.apply_S(x), padm.apply_S(x))}
    del x
    print(f"{name} {shape} vs port:", {k: f"{v:.2e}" for k, v in errs.items()})
    assert max(errs.values()) < OP_TOL, errs

    rhs = padm.build_rhs()[0]
    assert rel(drv.build_rhs()[0], rhs) < OP_TOL
    y_cpu, r_cpu = padm.pcg(rhs, tol=1e-8, max_inner=400)
    y_gpu, r_gpu = drv.pcg(rhs, tol=1e-8, max_inner=400)
    print(f"{name} PCG: gpu {r_gpu.iterations} its (rel res {r_gpu.rel_residual:.3e}), "
          f"port {r_cpu['iterations']} its (rel res {r_cpu['rel_residual']:.3e}); "
          f"|y_gpu - y_port| / |y_port| = {rel(y_gpu, y_cpu):.2e}")
    assert r_gpu.converged and abs(r_gpu.iterations - r_cpu["iterations"]) <= 1
    assert rel(y_gpu, y_cpu) < 1e-7
