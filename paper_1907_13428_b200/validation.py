"""Dense-oracle equivalence suite of the reference, Eigen-free (f4).

Restates fdeopt::oracle::run_validation (oracle.cpp:304-595) with numpy dense
assemblies (oracle.cpp:30-300: dense Toeplitz / circulant / Kronecker
constraint, 3-level T. Chan, preconditioned and normal-equation matrices,
the merged saddle solve of one ADMM step, the KKT residual) against a
structured backend: the B200 path (`B200Backend`, used by `cli validate` and
the GPU tests) or the C restatement in oracle/ (CPU CI gate, tests/).
Check names, order and thresholds are the reference's; the `perturb`
fault-injection hook perturbs one Caputo coefficient of the structured
operator only, so check 1 must fail (test_oracle.cpp:179-188).

Adaptations (the B200 interface differs, the property checked does not):
* random draws come from numpy's generator seeded with `seed`, not
  std::mt19937_64 (the checks are bounds, not golden values);
* check 2 runs the Toeplitz factor as the time factor of an (n, 1, 1)
  operator (the time factor is the one applied transposed by the adjoint);
* check 4 takes the eigenvalues of a circulant C as T. Chan's of the
  Toeplitz matrix C (T. Chan of a circulant is itself);
* check 5 compares the multiset lambda_S = rho (1 + 1/delta) + |lambda_B|^2 / m2
  (the preconditioner's exported spectrum) with the eigenvalues of the dense
  preconditioner rho (1 + 1/delta) I + C3^T C3 / m2.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DENSE_CAP = 6  # oracle.hpp kDenseCap


@dataclass
class CheckResult:
    name: str
    max_err: float
    threshold: float

    def passed(self) -> bool:
        return self.max_err <= self.threshold  # NaN fails


# ------------------------------------------------------------- dense side
def dense_toeplitz(col, row) -> np.ndarray:
    """oracle.cpp:30-36"""
    n = len(col)
    i, j = np.indices((n, n))
    return np.where(i >= j, np.asarray(col)[np.abs(i - j)], np.asarray(row)[np.abs(j - i)])


def dense_circulant(c) -> np.ndarray:
    """oracle.cpp:38-44"""
    n = len(c)
    i, j = np.indices((n, n))
    return np.asarray(c)[(i - j) % n]


def _factors(spec, n, perturb=0.0):
    from .api import build_caputo, build_riesz
    h = 1.0 / (n + 1)
    t = [np.array(a) for a in build_caputo(spec.alpha, n, h)]
    t[0][1 if n > 1 else 0] += perturb
    return t, build_riesz(spec.beta1, n, h), build_riesz(spec.beta2, n, h)


def dense_constraint(spec, n) -> np.ndarray:
    """oracle.cpp:54-64: psi (C (x) I (x) I - I (x) (L1 (x) I + I (x) L2))."""
    from .spec import scaling_psi
    t, r1, r2 = _factors(spec, n)
    e = np.eye(n)
    return scaling_psi(spec) * (np.kron(dense_toeplitz(*t), np.eye(n * n))
                                - np.kron(e, np.kron(dense_toeplitz(*r1), e) + np.kron(e, dense_toeplitz(*r2))))


def dense_c3(spec, n) -> np.ndarray:
    """oracle.cpp:66-75 (T. Chan circulant of each factor)."""
    from .api import tchan
    from .spec import scaling_psi
    t, r1, r2 = _factors(spec, n)
    ct, c1, c2 = (dense_circulant(tchan(*f)[0]) for f in (t, r1, r2))
    e = np.eye(n)
    return scaling_psi(spec) * (np.kron(ct, np.eye(n * n)) - np.kron(e, np.kron(c1, e) + np.kron(e, c2)))


def _m2(spec, rho, delta):
    from .spec import scaling_psi
    psi = scaling_psi(spec)
    return 1.0 / (rho * (spec.gamma / (psi * psi) + 1.0 / delta)) + delta / rho


def dense_precond(spec, n, rho, delta) -> np.ndarray:
    """oracle.cpp:77-85"""
    c3 = dense_c3(spec, n)
    return rho * (1.0 + 1.0 / delta) * np.eye(c3.shape[0]) + c3.T @ c3 / _m2(spec, rho, delta)


def _weights(spec, n):
    """objective_weights (problem.cpp:60-68) and J2 = (gamma/psi^2) J."""
    from .spec import scaling_psi
    j = np.ones(n ** 3)
    j[(n - 1) * n * n:] = 0.5
    psi = scaling_psi(spec)
    return j, spec.gamma / (psi * psi) * j


def dense_normal_matrix(spec, n, rho, delta, B) -> np.ndarray:
    """oracle.cpp:87-95 with the AdmmWork vectors of make_admm_work
    (admm.cpp:52-79): m2 = a2_inv + delta/rho, a2_inv = 1/(rho (J2 + 1/delta))."""
    j1, j2 = _weights(spec, n)
    m2 = 1.0 / (rho * (j2 + 1.0 / delta)) + delta / rho
    return np.diag(rho * (j1 + 1.0 / delta)) + B.T @ (B / m2[:, None])


@dataclass
class DenseProblem:
    """oracle.cpp:147-170"""
    B: np.ndarray
    psi: float
    j1: np.ndarray
    j2: np.ndarray
    ybar: np.ndarray
    delta: float
    rho: float
    y_lo: float
    y_hi: float
    v_lo: float
    v_hi: float


def make_dense_problem(spec, delta, rho) -> DenseProblem:
    from .spec import desired_state, scaling_psi
    n = spec.n
    j1, j2 = _weights(spec, n)
    psi = scaling_psi(spec)
    return DenseProblem(dense_constraint(spec, n), psi, j1, j2, desired_state(n), delta, rho, spec.y_lo,
                        spec.y_hi, psi * spec.u_lo, psi * spec.u_hi)


def dense_admm_step(dp: DenseProblem, s: dict) -> None:
    """oracle.cpp:179-216: the merged saddle system solved by LU."""
    N = dp.B.shape[0]
    rho, delta = dp.rho, dp.delta
    K = np.zeros((3 * N, 3 * N))
    K[:N, :N] = np.diag(rho * (dp.j1 + 1.0 / delta))
    K[:N, 2 * N:] = dp.B.T
    K[N:2 * N, N:2 * N] = np.diag(rho * (dp.j2 + 1.0 / delta))
    K[N:2 * N, 2 * N:] = np.eye(N)
    K[2 * N:, :N] = dp.B
    K[2 * N:, N:2 * N] = np.eye(N)
    K[2 * N:, 2 * N:] = -(delta / rho) * np.eye(N)
    rhs = np.concatenate([rho * (dp.j1 * dp.ybar - s["w_y"] + s["z_y"] / delta) + (1.0 - rho) * (dp.B.T @ s["p"]),
                          rho * (-s["w_v"] + s["z_v"] / delta) + (1.0 - rho) * s["p"],
                          -(delta / rho) * s["p"]])
    sol = np.linalg.solve(K, rhs)
    y, v, p = sol[:N], sol[N:2 * N], sol[2 * N:]
    s["y"], s["v"], s["p"] = y, v, p
    s["z_y"] = np.clip(y + delta * s["w_y"], dp.y_lo, dp.y_hi)
    s["z_v"] = np.clip(v + delta * s["w_v"], dp.v_lo, dp.v_hi)
    s["w_y"] = s["w_y"] + (rho / delta) * (y - s["z_y"])
    s["w_v"] = s["w_v"] + (rho / delta) * (v - s["z_v"])


def kkt_residual(dp: DenseProblem, s: dict) -> float:
    """max(stationarity, primal, bound violation) of oracle.cpp:246-276."""
    st_y = np.abs(dp.j1 * (s["y"] - dp.ybar) + dp.B.T @ s["p"] + s["w_y"]).max()
    st_v = np.abs(dp.j2 * s["v"] + s["p"] + s["w_v"]).max()
    primal = np.abs(dp.B @ s["y"] + s["v"]).max()
    bv = 0.0
    for z, lo, hi in ((s["z_y"], dp.y_lo, dp.y_hi), (s["z_v"], dp.v_lo, dp.v_hi)):
        if math.isfinite(lo):
            bv = max(bv, float((lo - z).max()))
        if math.isfinite(hi):
            bv = max(bv, float((z - hi).max()))
    return max(st_y, st_v, primal, max(bv, 0.0))


# ------------------------------------------------------ structured side
class B200Backend:
    """The B200 path through its public API (api.py)."""

    def __init__(self, ctx=None):
        from .api import default_context
        self.ctx = ctx or default_context()

    def op(self, time, x1, x2, psi, shape):
        from .api import ConstraintOperator
        return ConstraintOperator(time, x1, x2, psi, shape=shape, ctx=self.ctx)

    def precond(self, op, rho, delta, gamma):
        from .api import assemble_precond
        return assemble_precond(op, rho, delta, gamma)

    def tchan(self, col, row):
        from .api import tchan
        return tchan(col, row)

    def driver(self, spec, delta, rho, fixed_tol, max_inner, max_outer=500, tol_primal=1e-4):
        from .api import AdmmConfig, AdmmDriver
        from .spec import desired_state, scaling_psi
        op = self.spec_op(spec)
        pc = self.precond(op, rho, delta, spec.gamma)
        cfg = AdmmConfig(delta=delta, rho=rho, tol_primal=tol_primal, max_outer=max_outer, max_inner=max_inner,
                         fixed_krylov_tol=fixed_tol)
        d = AdmmDriver(op, pc, spec.gamma, cfg, y_lo=spec.y_lo, y_hi=spec.y_hi, u_lo=spec.u_lo, u_hi=spec.u_hi,
                       ybar=desired_state(spec.n))
        d._keep = (op, pc)
        d.scale_v = scaling_psi(spec)
        return d

    def spec_op(self, spec, perturb=0.0):
        from .spec import scaling_psi
        n = spec.n
        return self.op(*_factors(spec, n, perturb), scaling_psi(spec), (n, n, n))

    def solve_spec(self, spec, delta, rho, tol_primal, max_outer):
        from .spec import AdmmSettings, solve_spec
        return solve_spec(spec, AdmmSettings(delta=delta, rho=rho, tol_primal=tol_primal, max_outer=max_outer),
                          ctx=self.ctx, keep_state=True)


# ----------------------------------------------------------------- suite
def run_validation(backend, cap: int = 4, perturb: float = 0.0, seed: int = 1):
    """oracle.cpp:304-595"""
    from .spec import ConfigError, ProblemSpec, scaling_psi
    if cap < 1 or cap > DENSE_CAP:
        raise ConfigError("run_validation: cap must lie in [1, 6]")
    rng = np.random.default_rng(seed)
    res = []

    def vspec(n, **kw):
        return ProblemSpec(n=n, alpha=0.7, beta1=1.3, beta2=1.3, gamma=1e-4, **kw)

    # 1. structured apply vs dense Kronecker assembly on the unit basis
    err = 0.0
    for n in range(1, cap + 1):
        for alpha in (0.5, 0.7):
            b = 1.5 if alpha == 0.5 else 1.3
            spec = ProblemSpec(n=n, alpha=alpha, beta1=b, beta2=b, gamma=1e-4)
            op = backend.spec_op(spec, perturb)
            dense = dense_constraint(spec, n)
            scale = np.abs(dense).max()
            cols = np.stack([op.apply(e) for e in np.eye(n ** 3)], axis=1)
            err = max(err, float(np.abs(cols - dense).max() / scale))
    res.append(CheckResult("matvec_unit_basis", err, 1e-13))

    # 2. FFT Toeplitz matvec vs dense, including transposes
    err = 0.0
    for n in (1, 2, 3, 5, 8):
        col, row = rng.standard_normal(n), rng.standard_normal(n)
        row[0] = col[0]
        T = dense_toeplitz(col, row)
        x = rng.standard_normal(n)
        z = (np.zeros(1), np.zeros(1))
        op = backend.op((col, row), z, z, 1.0, (n, 1, 1))
        for tr in (False, True):
            want = (T.T if tr else T) @ x
            got = op.apply(x, tr)
            err = max(err, float(np.abs(got - want).max() / max(1.0, np.abs(want).max())))
    res.append(CheckResult("toeplitz_matvec_dense", err, 1e-12))

    # 3. T. Chan optimality (Frobenius) and diagonal averaging
    gap = 0.0
    for _ in range(50):
        n = int(rng.integers(1, 9))
        col, row = rng.standard_normal(n), rng.standard_normal(n)
        row[0] = col[0]
        T = dense_toeplitz(col, row)
        c = backend.tchan(col, row)[0]
        best = np.linalg.norm(dense_circulant(c) - T)
        cands = rng.standard_normal((200, n))
        for cand in cands:
            gap = max(gap, float(best - np.linalg.norm(dense_circulant(cand) - T)))
        for i in range(n):
            acc = sum(T[(r + i) % n, r] for r in range(n))
            gap = max(gap, abs(acc / n - c[i]))
    res.append(CheckResult("tchan_frobenius", gap, 1e-12))

    # 4. circulant eigen-identity against dense Fourier vectors
    err = 0.0
    for n in (2, 3, 7, 16, 32):
        c = rng.standard_normal(n)
        row = np.concatenate([[c[0]], c[1:][::-1]])
        eigs = backend.tchan(c, row)[1]
        C = dense_circulant(c)
        k = np.arange(n)
        for j in range(n):
            xj = np.exp(2j * np.pi * j * k / n)
            err = max(err, float(np.abs(C @ xj - eigs[j] * xj).max() / max(1.0, abs(eigs[j]))))
    res.append(CheckResult("circulant_eigen_identity", err, 1e-12))

    # 5. preconditioner spectrum vs the dense 3-level assembly
    err = 0.0
    for n in range(1, min(cap, 4) + 1):
        spec = vspec(n)
        pc = backend.precond(backend.spec_op(spec), 1.618, 2.0, spec.gamma)
        want = np.sort(np.linalg.eigvalsh(dense_precond(spec, n, 1.618, 2.0)))
        got = np.sort(pc.lam_s())
        err = max(err, float(np.abs(got - want).max() / max(1.0, np.abs(want).max())))
    res.append(CheckResult("precond_eigs_multiset", err, 1e-10))

    # 6. preconditioner solve vs dense solve
    err = 0.0
    for n in range(1, min(cap, 4) + 1):
        spec = vspec(n)
        pc = backend.precond(backend.spec_op(spec), 1.618, 0.4, spec.gamma)
        r = rng.standard_normal(n ** 3)
        z = pc.solve(r)
        err = max(err, float(np.linalg.norm(dense_precond(spec, n, 1.618, 0.4) @ z - r) / np.linalg.norm(r)))
    res.append(CheckResult("precond_solve_dense", err, 1e-12))

    # 7. apply_S vs the dense normal-equations matrix
    err = 0.0
    for n in range(2, min(cap, 4) + 1):
        spec = vspec(n)
        drv = backend.driver(spec, 2.0, 1.618, 1e-8, 400)
        S = dense_normal_matrix(spec, n, 1.618, 2.0, dense_constraint(spec, n))
        x = rng.standard_normal(n ** 3)
        want = S @ x
        err = max(err, float(np.abs(drv.apply_S(x) - want).max() / max(1.0, np.abs(want).max())))
    res.append(CheckResult("apply_s_dense", err, 1e-12))

    # 8. one structured step (tight inner solve) satisfies the merged block
    #    system of its start state
    n = min(cap, 3)
    if n >= 1:
        spec = vspec(n)
        N = n ** 3
        drv = backend.driver(spec, 2.0, 1.618, 1e-14, 10 * N)
        st = {k: rng.standard_normal(N) for k in ("z_y", "z_v", "p", "w_y", "w_v")}
        for k, v in st.items():
            drv.set(k, v)
        drv.step()
        y, v, p = drv.get("y"), drv.get("v"), drv.get("p")
        rho, delta = 1.618, 2.0
        B = dense_constraint(spec, n)
        j1, j2 = _weights(spec, n)
        from .spec import desired_state
        ybar = desired_state(n)
        r1 = rho * (j1 + 1.0 / delta) * y + B.T @ p - (rho * (j1 * ybar - st["w_y"] + st["z_y"] / delta)
                                                      + (1.0 - rho) * (B.T @ st["p"]))
        r2 = rho * (j2 + 1.0 / delta) * v + p - (rho * (-st["w_v"] + st["z_v"] / delta) + (1.0 - rho) * st["p"])
        r3 = B @ y + v - (delta / rho) * p + (delta / rho) * st["p"]
        rhs_scale = max(1.0, float(np.abs(rho * (j1 * ybar - st["w_y"] + st["z_y"] / delta)).max()))
        res.append(CheckResult("saddle_recovery_residual",
                               max(np.abs(r1).max(), np.abs(r2).max(), np.abs(r3).max()) / rhs_scale, 1e-10))

    # 9. five structured ADMM iterations vs the dense factorized route
    err = 0.0
    for n in range(2, min(cap, 4) + 1, 2):
        spec = vspec(n)
        N = n ** 3
        drv = backend.driver(spec, 0.4, 1.618, 1e-14, 10 * N)
        dp = make_dense_problem(spec, 0.4, 1.618)
        ds = {k: np.zeros(N) for k in ("y", "v", "z_y", "z_v", "p", "w_y", "w_v")}
        for k in ("z_y", "z_v", "p", "w_y", "w_v"):
            ds[k] = rng.standard_normal(N)
            drv.set(k, ds[k])
        for _ in range(5):
            drv.step()
            dense_admm_step(dp, ds)
            for k in ("y", "v", "p", "z_y", "z_v", "w_y", "w_v"):
                err = max(err, float(np.abs(drv.get(k) - ds[k]).max()))
    res.append(CheckResult("admm_dense_equivalence", err, 1e-10))

    # 10. the unconstrained ADMM limit satisfies the dense KKT system
    n = min(cap, 4)
    spec = vspec(n)
    out = backend.solve_spec(spec, 2.0, 1.618, 1e-5, 3000)
    dp = make_dense_problem(spec, 2.0, 1.618)
    s = {k: out[k] for k in ("y", "z_y", "z_v", "p", "w_y", "w_v")}
    s["v"] = scaling_psi(spec) * out["u"]
    res.append(CheckResult("unconstrained_kkt", kkt_residual(dp, s), 1e-3))
    return res


def format_report(results) -> str:
    """cmd_validate's table (fdeopt_main.cpp:197-208)."""
    from .io import fmt_g
    lines = ["%-28s %-14s %-10s %s" % ("check", "max_err", "threshold", "result")]
    for r in results:
        lines.append("%-28s %-14s %-10s %s" % (r.name, fmt_g(r.max_err), fmt_g(r.threshold),
                                                "PASS" if r.passed() else "FAIL"))
    return "\n".join(lines)
