"""Full ADMM solves of the BASELINE C2, C3 and C4 problem structures (their
formulas, bounds, orders and regularisation; grid reduced to 8 x 16 x 16 so
the C restatement of the reference finishes in seconds) on the B200 path vs
the oracle: the same ADMM step count, the same Krylov count on every step
(+-1 allowed by the north star), final iterate and objective within 1e-8."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPE = (8, 16, 16)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_full_solve_vs_oracle(gpu_ctx, port, name):
    from oracle import Shape, baseline_problem
    from oracle.pyoracle import PortAdmm
    from paper_1907_13428_b200 import AdmmConfig, AdmmDriver, ConstraintOperator, assemble_precond
    from paper_1907_13428_b200.workloads import synthetic_ybar
    c = baseline_problem(name, Shape(*SHAPE))
    yb = synthetic_ybar(c["ybar"], SHAPE)
    pop = port.op(SHAPE, c["time"], c["r1"], c["r2"], c["psi"])
    ppc = pop.assemble_precond(1.0, 1.0, c["gamma"])
    padm = PortAdmm(port, pop, ppc, c["gamma"], 1.0, 1.0, y_lo=c["y"][0], y_hi=c["y"][1], u_lo=c["u"][0],
                    u_hi=c["u"][1], tol_primal=1e-6, max_inner=400, fixed_tol=1e-8, ybar=yb)
    op = ConstraintOperator(c["time"], c["r1"], c["r2"], c["psi"], shape=SHAPE, ctx=gpu_ctx)
    pc = assemble_precond(op, 1.0, 1.0, c["gamma"])
    cfg = AdmmConfig(delta=1.0, rho=1.0, tol_primal=1e-6, max_outer=20000, max_inner=400, fixed_krylov_tol=1e-8)
    drv = AdmmDriver(op, pc, c["gamma"], cfg, y_lo=c["y"][0], y_hi=c["y"][1], u_lo=c["u"][0], u_hi=c["u"][1],
                     ybar=yb)
    inner_gpu, inner_cpu = [], []
    for _ in range(20000):
        g, p = drv.step(), padm.step()
        inner_gpu.append(g.inner_iters)
        inner_cpu.append(p["inner_iters"])
        assert g.converged == p["converged"], len(inner_gpu)
        if g.converged:
            break
    assert drv.converged() and len(inner_gpu) > 100
    d = np.abs(np.array(inner_gpu) - np.array(inner_cpu))
    assert d.max() <= 1, (int(d.max()), int((d > 0).sum()))
    for f in ("y", "v", "p"):
        assert rel(drv.get(f), padm.get(f)) < 1e-8, f
    assert abs(drv.objective() - padm.objective()) <= 1e-8 * abs(padm.objective())
    assert abs(drv.dual_infeasibility() - padm.dual_inf()) <= 1e-8 * abs(padm.dual_inf()) + 1e-14
