"""GPU parity of the sm_100a path against the CPU oracle (unchanged reference
in oracle/_ref and the generalized C restatement in oracle/build).

Tolerances (BASELINE.json north_star): operator / preconditioner 1e-11
relative (2-norm, as SURVEY.md App. A.9); PCG iteration counts +-1; ADMM
residuals / objective 1e-8 relative.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

OP_TOL = 1e-11


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def gpu_op(ctx, time, x1, x2, psi):
    from paper_1907_13428_b200 import ConstraintOperator
    return ConstraintOperator(time, x1, x2, psi, ctx=ctx)


# ------------------------------------------------------------ operator
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 16, 17, 32])
def test_operator_reference_default_spec(gpu_ctx, ref, n):
    """ConstraintOperator(spec, grid) with the reference defaults (Caputo
    alpha=0.7 time factor -> FFT time pass), vs the unchanged reference."""
    rop = ref.op_spec(0.7, 1.3, 1.3, n)
    h = 1.0 / (n + 1)
    t = ref.build_caputo(0.7, n, h)
    r1 = ref.build_riesz(1.3, n, h)
    r2 = ref.build_riesz(1.3, n, h)
    op = gpu_op(gpu_ctx, t, r1, r2, rop.psi)
    x = ref.randn(7 + n, n ** 3)
    for adj in (False, True):
        assert rel(op.apply(x, adj), rop.apply(x, adj)) < OP_TOL


@pytest.mark.parametrize("n", [4, 8, 16])
def test_operator_golden(gpu_ctx, ref, golden, n):
    from oracle import Shape, baseline_problem
    c = baseline_problem("C0", Shape(n, n, n))
    op = gpu_op(gpu_ctx, c["time"], c["r1"], c["r2"], c["psi"])
    x = golden[f"ie{n}_x"]
    assert rel(op.apply(x, False), golden[f"ie{n}_Bx"]) < OP_TOL
    assert rel(op.apply(x, True), golden[f"ie{n}_BTx"]) < OP_TOL


@pytest.mark.parametrize("shape", [(4, 8, 16), (16, 8, 4), (3, 5, 7), (32, 64, 64), (8, 128, 32),
                                   (2, 256, 256), (1, 33, 47), (2, 16, 512), (2, 512, 16),
                                   (2, 8, 1024), (2, 1024, 8), (2, 300, 700)])
def test_operator_noncube_vs_port(gpu_ctx, port, shape):
    """Non-cube shapes (BASELINE C1/C3/C4 structure) against the generalized
    C restatement, anisotropic orders and diffusion coefficients."""
    from oracle import implicit_euler
    nt, n1, n2 = shape
    t = implicit_euler(nt, 1.0 / nt)
    c1 = port.build_riesz(1.8, n1, 1.0 / (n1 + 1))
    c2 = port.build_riesz(1.2, n2, 1.0 / (n2 + 1))
    c1 = (c1[0] * 0.5, c1[1] * 0.5)
    psi = min(1.0 / nt, (1.0 / (n2 + 1)) ** 1.2, (1.0 / (n1 + 1)) ** 1.8)
    pop = port.op(shape, t, c1, c2, psi)
    op = gpu_op(gpu_ctx, t, c1, c2, psi)
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(nt * n1 * n2)
    for adj in (False, True):
        assert rel(op.apply(x, adj), pop.apply(x, adj)) < OP_TOL


def test_operator_size_check(gpu_ctx, ref):
    n = 2
    op = gpu_op(gpu_ctx, ref.build_caputo(0.7, n, 1 / 3), ref.build_riesz(1.3, n, 1 / 3),
                ref.build_riesz(1.3, n, 1 / 3), 0.1)
    with pytest.raises(ValueError):
        op.apply(np.zeros(3))


def test_operator_adjoint_identity_large(gpu_ctx):
    """<Bx, y> == <x, B^T y> at a BASELINE-size slab (size-independent property)."""
    from paper_1907_13428_b200 import baseline_config, randn
    c = baseline_config("C2", (64, 256, 256))
    op = gpu_op(gpu_ctx, c["time"], c["x1"], c["x2"], c["psi"])
    x = randn(3, op.size)
    y = randn(4, op.size)
    bx = op.apply(x)
    bty = op.apply(y, True)
    a, b = bx @ y, x @ bty
    assert abs(a - b) <= 1e-12 * np.abs(bx * y).sum()


# ------------------------------------------------------ preconditioner
# 3, 5, 6, 12, 17: level sizes without a radix plan take the dense Hartley path
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 8, 12, 16, 17, 32])
def test_precond_reference_default(gpu_ctx, ref, n):
    from paper_1907_13428_b200 import assemble_precond
    rop = ref.op_spec(0.7, 1.3, 1.3, n)
    rpc = rop.assemble_precond(1.618, 0.4, 1e-4)
    h = 1.0 / (n + 1)
    op = gpu_op(gpu_ctx, ref.build_caputo(0.7, n, h), ref.build_riesz(1.3, n, h),
                ref.build_riesz(1.3, n, h), rop.psi)
    pc = assemble_precond(op, 1.618, 0.4, 1e-4)
    x = ref.randn(11 + n, n ** 3)
    assert rel(pc.solve(x), rpc.solve(x)) < OP_TOL
    assert rel(pc.lam_s(), rpc.lam_s()) < 1e-13


@pytest.mark.parametrize("n", [4, 8, 16])
def test_precond_golden(gpu_ctx, golden, n):
    from oracle import Shape, baseline_problem
    from paper_1907_13428_b200 import assemble_precond
    c = baseline_problem("C0", Shape(n, n, n))
    op = gpu_op(gpu_ctx, c["time"], c["r1"], c["r2"], c["psi"])
    pc = assemble_precond(op, 1.0, 1.0, c["gamma"])
    assert rel(pc.solve(golden[f"ie{n}_x"]), golden[f"ie{n}_Minv_x"]) < OP_TOL


@pytest.mark.parametrize("shape", [(4, 8, 16), (16, 8, 4), (32, 64, 64), (8, 128, 32), (1, 32, 64),
                                   # n1 == n2 in {256, 512}: x2/x1 pairs fused through L2, fewer
                                   # and more slabs than the pipeline lag
                                   (1, 256, 256), (4, 256, 256), (32, 256, 256), (2, 512, 512),
                                   (16, 512, 512),
                                   # n_t = 128 / 256: the t filters k_t_filter<128|256> of the
                                   # timed C3/C4 and C2 configs
                                   (128, 16, 32), (256, 16, 16), (128, 64, 64), (256, 32, 64)])
def test_precond_noncube_vs_port(gpu_ctx, port, shape):
    from oracle import implicit_euler
    from paper_1907_13428_b200 import assemble_precond
    nt, n1, n2 = shape
    t = implicit_euler(nt, 1.0 / nt)
    c1 = port.build_riesz(1.8, n1, 1.0 / (n1 + 1))
    c2 = port.build_riesz(1.2, n2, 1.0 / (n2 + 1))
    psi = min(1.0 / nt, (1.0 / (n2 + 1)) ** 1.2, (1.0 / (n1 + 1)) ** 1.8)
    pop = port.op(shape, t, c1, c2, psi)
    ppc = pop.assemble_precond(1.0, 1.0, 1e-6)
    op = gpu_op(gpu_ctx, t, c1, c2, psi)
    pc = assemble_precond(op, 1.0, 1.0, 1e-6)
    x = np.random.default_rng(5).standard_normal(op.size)
    assert rel(pc.solve(x), ppc.solve(x)) < OP_TOL


def test_precond_identity_and_halving(gpu_ctx, ref):
    """test_circulant.cpp:139-155: lambda_B == 0 -> rho(1+1/delta) scaling."""
    from paper_1907_13428_b200 import CirculantPreconditioner
    z = np.zeros(4, dtype=complex)
    r = ref.randn(31, 64)
    ident = CirculantPreconditioner.from_eigs(z, z, z, 1.0, 0.5, 1.0, 1e-4, ctx=gpu_ctx)
    assert np.allclose(ident.solve(r), r, rtol=1e-13, atol=1e-14)
    half = CirculantPreconditioner.from_eigs(z, z, z, 1.0, 1.0, 1.0, 1e-4, ctx=gpu_ctx)
    assert np.allclose(half.solve(r), r / 2.0, rtol=1e-13, atol=1e-14)
    with pytest.raises(ValueError):
        half.solve(np.zeros(5))


# ------------------------------------------------------------ S / PCG
def _drivers(gpu_ctx, ref, n, ybar=None):
    from oracle import Shape, baseline_problem, synthetic_ybar
    from oracle.pyoracle import RefAdmm
    from paper_1907_13428_b200 import AdmmConfig, AdmmDriver, assemble_precond
    c = baseline_problem("C0", Shape(n, n, n))
    yb = synthetic_ybar("sin", Shape(n, n, n)) if ybar is None else ybar
    rop = ref.op(n, c["time"], c["r1"], c["r2"], c["psi"])
    rpc = rop.assemble_precond(1.0, 1.0, c["gamma"])
    radm = RefAdmm(ref, rop, rpc, c["gamma"], 1.0, 1.0, u_lo=c["u"][0], u_hi=c["u"][1],
                   tol_primal=1e-6, max_inner=400, fixed_tol=1e-8, ybar=yb)
    op = gpu_op(gpu_ctx, c["time"], c["r1"], c["r2"], c["psi"])
    pc = assemble_precond(op, 1.0, 1.0, c["gamma"])
    cfg = AdmmConfig(delta=1.0, rho=1.0, tol_primal=1e-6, max_outer=100000, max_inner=400,
                     fixed_krylov_tol=1e-8)
    drv = AdmmDriver(op, pc, c["gamma"], cfg, u_lo=c["u"][0], u_hi=c["u"][1], ybar=yb)
    return radm, drv


@pytest.mark.parametrize("n", [4, 8, 16])
def test_apply_S_and_rhs(gpu_ctx, ref, golden, n):
    radm, drv = _drivers(gpu_ctx, ref, n, golden[f"ie{n}_ybar"])
    x = golden[f"ie{n}_x"]
    assert rel(drv.apply_S(x), golden[f"ie{n}_Sx"]) < OP_TOL
    rhs, _ = drv.build_rhs()
    assert rel(rhs, golden[f"ie{n}_rhs0"]) < OP_TOL
    y, res = drv.pcg(rhs, tol=1e-8, max_inner=400)
    assert abs(res.iterations - int(golden[f"ie{n}_pcg0_iters"][0])) <= 1
    assert rel(y, golden[f"ie{n}_pcg0_y"]) < 1e-8


@pytest.mark.parametrize("n", [4, 8, 16])
def test_admm_five_steps_golden(gpu_ctx, ref, golden, n):
    _, drv = _drivers(gpu_ctx, ref, n, golden[f"ie{n}_ybar"])
    inner = []
    res = []
    for _ in range(5):
        r = drv.step()
        inner.append(r.inner_iters)
        res.append([r.r_eq, r.r_y, r.r_u, r.dual_inf])
    want = golden[f"ie{n}_steps_inner"]
    assert np.all(np.abs(np.array(inner) - want) <= 1), (inner, want)
    got, exp = np.array(res), golden[f"ie{n}_steps_res"]
    mask = exp > 1e-12
    assert np.all(np.abs(got[mask] - exp[mask]) <= 1e-8 * np.abs(exp[mask]) + 1e-14)
    for f in ("y", "v", "p"):
        assert rel(drv.get(f), golden[f"ie{n}_after5_{f}"]) < 1e-8
    assert abs(drv.objective() - golden[f"ie{n}_after5_obj"][0]) <= 1e-8 * abs(golden[f"ie{n}_after5_obj"][0])


@pytest.mark.parametrize("shape", [(4, 16, 256), (4, 8, 512), (2, 16, 64), (2, 4, 1024),
                                   # n1 = 256 / 512 / 1024: the split S-mid column passes
                                   # k_colc<512|1024|2048, 2> the bench times (K2) and the
                                   # staged row passes k_rowc<512> / k_rowq<1024> / k_rowc<2048>
                                   (2, 256, 256), (2, 512, 64), (2, 1024, 32), (2, 16, 1024),
                                   (2, 512, 512),
                                   # more tiles than resident CTAs: the persistent loops'
                                   # staging / prefetch across tiles
                                   (24, 256, 256), (8, 512, 256)])
def test_pcg_noncube_vs_port(gpu_ctx, port, shape):
    """PCG on the ADMM normal equations for shapes that select the staged
    row kernels (tiles inside one slice), the L >= 1024 single-buffer
    kernels and the split column passes of the timed configs, against the
    generalized C restatement: S within 1e-11, Krylov count +-1."""
    from oracle import Shape, baseline_problem
    from oracle.pyoracle import PortAdmm
    from paper_1907_13428_b200 import AdmmConfig, AdmmDriver, assemble_precond
    c = baseline_problem("C3", Shape(*shape))
    pop = port.op(shape, c["time"], c["r1"], c["r2"], c["psi"])
    ppc = pop.assemble_precond(1.0, 1.0, c["gamma"])
    rng = np.random.default_rng(11)
    yb = rng.standard_normal(pop.size)
    padm = PortAdmm(port, pop, ppc, c["gamma"], 1.0, 1.0, y_lo=c["y"][0], y_hi=c["y"][1],
                    u_lo=c["u"][0], u_hi=c["u"][1], tol_primal=1e-6, max_inner=400,
                    fixed_tol=1e-8, ybar=yb)
    op = gpu_op(gpu_ctx, c["time"], c["r1"], c["r2"], c["psi"])
    pc = assemble_precond(op, 1.0, 1.0, c["gamma"])
    cfg = AdmmConfig(delta=1.0, rho=1.0, tol_primal=1e-6, max_inner=400, fixed_krylov_tol=1e-8)
    drv = AdmmDriver(op, pc, c["gamma"], cfg, y_lo=c["y"][0], y_hi=c["y"][1], u_lo=c["u"][0],
                     u_hi=c["u"][1], ybar=yb)
    x = rng.standard_normal(pop.size)
    assert rel(drv.apply_S(x), padm.apply_S(x)) < OP_TOL
    rhs = padm.build_rhs()[0]
    assert rel(drv.build_rhs()[0], rhs) < OP_TOL
    y_cpu, r_cpu = padm.pcg(rhs, tol=1e-8, max_inner=400)
    y_gpu, r_gpu = drv.pcg(rhs, tol=1e-8, max_inner=400)
    assert r_gpu.converged and abs(r_gpu.iterations - r_cpu["iterations"]) <= 1
    assert rel(y_gpu, y_cpu) < 1e-7
    for _ in range(2):
        g, cpu = drv.step(), padm.step()
        assert abs(g.inner_iters - cpu["inner_iters"]) <= 1


@pytest.mark.parametrize("x0_kind", ["zero", "negzero", "warm", "one_nonzero"])
def test_pcg_host_x0_paths(gpu_ctx, ref, golden, x0_kind):
    """fdg_admm_pcg_host speculates on x0 = 0 while x0 is in flight and redoes
    the solve from x0 otherwise: its result must equal the device-buffer path
    (fdg_admm_pcg) from the same x0 bit for bit, with the same count."""
    import torch
    n = 8
    _, drv = _drivers(gpu_ctx, ref, n, golden[f"ie{n}_ybar"])
    rhs, _ = drv.build_rhs()
    N = rhs.size
    x0 = np.zeros(N)
    if x0_kind == "negzero":
        x0[:] = -0.0
    elif x0_kind == "warm":
        x0 = golden[f"ie{n}_pcg0_y"] * 0.9
    elif x0_kind == "one_nonzero":
        x0[N - 1] = 1e-3
    xh = x0.copy()
    _, r_host = drv.pcg(rhs, xh, tol=1e-8, max_inner=400)
    rhs_d = torch.tensor(rhs, dtype=torch.float64, device="cuda")
    x_d = torch.tensor(x0, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    r_dev = drv.pcg_dev(rhs_d, x_d, 1e-8, 400)
    torch.cuda.synchronize()
    assert r_host.iterations == r_dev.iterations
    assert np.array_equal(xh, x_d.cpu().numpy())


@pytest.mark.parametrize("shape", [(32, 32, 32), (8, 16, 64), (5, 12, 16)])
def test_pcg_graph_iterations_match_host_sequenced(gpu_ctx, shape):
    """The graph-driven PCG iterations (one CUDA graph launch per solve, a
    WHILE node stopped by the device control step) run the same kernels in
    the same order as the host-sequenced loop: identical Krylov counts and
    bitwise-identical solutions, for converged solves, the max_inner cap
    (both parities of the stopping iteration) and whole ADMM steps."""
    import torch
    from paper_1907_13428_b200 import make_problem
    from paper_1907_13428_b200.api import set_pcg_graph_nmax
    out = {}
    prev = set_pcg_graph_nmax(0)
    try:
        for mode, nmax in (("host", 0), ("graph", 1 << 40)):
            set_pcg_graph_nmax(nmax)
            c, op, pc, drv = make_problem("C0", shape, ctx=gpu_ctx)
            rhs, _ = drv.build_rhs()
            rhs_d = torch.tensor(rhs, device="cuda")
            runs = []
            for tol, cap in ((1e-8, 400), (1e-30, 5), (1e-30, 6), (1e-30, 1)):
                x = torch.zeros_like(rhs_d)
                torch.cuda.synchronize()
                r = drv.pcg_dev(rhs_d, x, tol, cap)
                torch.cuda.synchronize()
                runs.append((r.iterations, r.converged, r.rel_residual, x.cpu().numpy()))
            recs = [drv.step() for _ in range(4)]
            runs.append([(s.inner_iters, s.r_eq, s.r_y, s.r_u, s.dual_inf) for s in recs])
            runs.append(drv.get("y"))
            out[mode] = runs
    finally:
        set_pcg_graph_nmax(prev)
    h, g = out["host"], out["graph"]
    for a, b in zip(h[:4], g[:4]):
        assert a[:3] == b[:3]
        assert np.array_equal(a[3], b[3])
    assert h[0][0] > 4 and h[1][0] == 5 and h[2][0] == 6
    assert h[4] == g[4]
    assert np.array_equal(h[5], g[5])
