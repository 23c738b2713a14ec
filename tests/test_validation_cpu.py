"""The reference's dense-oracle equivalence suite (oracle.cpp:304-595),
restated without Eigen (paper_1907_13428_b200/validation.py), as a CI gate in
this GPU-less container (f4): run against the C restatement of
the hot path (oracle/), every check passes; with the fault-injection hook
(--perturb) the unit-basis check fails (test_oracle.cpp:179-188)."""
import math

import numpy as np
import pytest

from paper_1907_13428_b200.validation import (CheckResult, DENSE_CAP, dense_circulant, dense_toeplitz,
                                              format_report, run_validation)

NAMES = ["matvec_unit_basis", "toeplitz_matvec_dense", "tchan_frobenius", "circulant_eigen_identity",
         "precond_eigs_multiset", "precond_solve_dense", "apply_s_dense", "saddle_recovery_residual",
         "admm_dense_equivalence", "unconstrained_kkt"]


class PortBackend:
    """validation's structured side on the oracle's C restatement."""

    def __init__(self):
        from oracle import port_lib
        self.P = port_lib()

    def op(self, time, x1, x2, psi, shape):
        return self.P.op(shape, time, x1, x2, psi)

    def precond(self, op, rho, delta, gamma):
        return op.assemble_precond(rho, delta, gamma)

    def tchan(self, col, row):
        return self.P.tchan(col, row)

    def spec_op(self, spec, perturb=0.0):
        from paper_1907_13428_b200.spec import scaling_psi
        from paper_1907_13428_b200.validation import _factors
        n = spec.n
        return self.op(*_factors(spec, n, perturb), scaling_psi(spec), (n, n, n))

    def driver(self, spec, delta, rho, fixed_tol, max_inner, max_outer=500, tol_primal=1e-4):
        from oracle.pyoracle import PortAdmm
        from paper_1907_13428_b200.spec import desired_state
        op = self.spec_op(spec)
        pc = self.precond(op, rho, delta, spec.gamma)
        return PortAdmm(self.P, op, pc, spec.gamma, rho, delta, y_lo=spec.y_lo, y_hi=spec.y_hi,
                        u_lo=spec.u_lo, u_hi=spec.u_hi, tol_primal=tol_primal, max_inner=max_inner,
                        fixed_tol=fixed_tol, ybar=desired_state(spec.n))

    def solve_spec(self, spec, delta, rho, tol_primal, max_outer):
        """fdeopt::solve's loop (admm.cpp:289-324) over the port driver,
        with the reference's dynamic inner tolerance."""
        from paper_1907_13428_b200.spec import scaling_psi
        d = self.driver(spec, delta, rho, 0.0, 400, max_outer, tol_primal)
        for _ in range(max_outer):
            if d.step()["converged"]:
                break
        out = {k: d.get(k) for k in ("y", "p", "w_y", "w_v", "z_y", "z_v")}
        out["u"] = d.get("v") / scaling_psi(spec)
        return out


@pytest.fixture(scope="module")
def port_results():
    return run_validation(PortBackend(), cap=4, perturb=0.0, seed=1)


def test_suite_passes_on_the_restatement(port_results):
    assert [r.name for r in port_results] == NAMES
    bad = [r for r in port_results if not r.passed()]
    assert not bad, format_report(port_results)


def test_fault_injection_is_detected():
    res = run_validation(PortBackend(), cap=2, perturb=1e-6, seed=3)
    by = {r.name: r for r in res}
    assert not by["matvec_unit_basis"].passed()
    assert all(r.passed() for r in res if r.name != "matvec_unit_basis"), format_report(res)


def test_dense_helpers_and_report():
    T = dense_toeplitz([1.0, 2.0, 3.0], [1.0, -1.0, -2.0])
    assert np.array_equal(T, [[1, -1, -2], [2, 1, -1], [3, 2, 1]])
    assert np.array_equal(dense_circulant([1.0, 2.0, 3.0]), [[1, 3, 2], [2, 1, 3], [3, 2, 1]])
    rep = format_report([CheckResult("x", 1e-15, 1e-13), CheckResult("y", math.nan, 1.0)]).splitlines()
    assert rep[0].split() == ["check", "max_err", "threshold", "result"]
    assert rep[1].split() == ["x", "1e-15", "1e-13", "PASS"] and rep[2].split()[-1] == "FAIL"
    from paper_1907_13428_b200.spec import ConfigError
    with pytest.raises(ConfigError, match=r"cap must lie in \[1, 6\]"):
        run_validation(PortBackend(), cap=DENSE_CAP + 1)
