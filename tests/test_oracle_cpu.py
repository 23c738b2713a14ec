"""The CPU oracle pinned before it is trusted.

* Known-answer vectors from the reference's own unit tests, asserted on both
  the unchanged reference (oracle/_ref) and the C restatement (oracle/build).
* The restatement against the unchanged reference on cube sizes (bitwise for
  shared FFT code paths; 1e-13 otherwise) and against direct O(n^2) sums.
* The committed golden fixtures (tests/golden/ref_small.npz, generated from
  oracle/_ref by tests/golden/make_golden.py) against a live run.
* The fault-injection fixture: a one-coefficient perturbation is detected.
"""
import math
import os

import numpy as np
import pytest

from oracle import Shape, baseline_problem, implicit_euler, synthetic_ybar

HERE = os.path.dirname(os.path.abspath(__file__))


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def dense_toeplitz(col, row):
    n = len(col)
    return np.array([[col[i - j] if i >= j else row[j - i] for j in range(n)] for i in range(n)])


# -------------------------------------------------- known answers (§8c table)
def test_frac_coeffs_known_answers(ref, port):
    for lib in (ref, port):
        assert np.allclose(lib.frac_coeffs(0.7, 3), [1.0, -0.7, -0.105], rtol=1e-14)  # test_problem.cpp:31-34
        assert np.allclose(lib.frac_coeffs(1.3, 3), [1.0, -1.3, 0.195], rtol=1e-14)   # 35-38
        assert list(lib.frac_coeffs(0.42, 1)) == [1.0]
        with pytest.raises(ValueError):
            lib.frac_coeffs(1.0, 4)
        with pytest.raises(ValueError):
            lib.frac_coeffs(0.5, 0)


def test_frac_coeffs_gamma_oracle(ref):
    """test_problem.cpp:16-50: agreement with the lgamma closed form to 1e-10."""
    def gamma_formula(c, k):
        def sg(x):
            return 1.0 if x > 0 else (1.0 if math.floor(x) % 2 == 0 else -1.0)
        return sg(k - c) * sg(-c) * math.exp(math.lgamma(k - c) - math.lgamma(-c) - math.lgamma(k + 1.0))
    for c in (0.1, 0.3, 0.7, 0.95, 1.05, 1.3, 1.5, 1.9):
        g = ref.frac_coeffs(c, 51)
        want = np.array([gamma_formula(c, k) for k in range(51)])
        assert np.allclose(g, want, rtol=1e-10, atol=0)


def test_caputo_riesz_known_answers(ref, port):
    for lib in (ref, port):
        col, row = lib.build_caputo(0.5, 3, 1.0)          # test_toeplitz.cpp:33-35
        assert list(col) == [1.0, -0.5, -0.125] and list(row) == [1.0, 0.0, 0.0]
        col, _ = lib.build_caputo(0.7, 2, 0.5)            # 40-42
        assert col[0] == pytest.approx(1.62450, rel=1e-5) and col[1] == pytest.approx(-1.13715, rel=1e-5)
        one, _ = lib.build_riesz(1.3, 1, 1.0)             # 50-53
        assert one[0] == pytest.approx(-2.8635, rel=1e-4)
        two, _ = lib.build_riesz(1.5, 2, 1.0)             # 56-60
        assert two[0] == pytest.approx(-3 / math.sqrt(2), rel=1e-14)
        assert two[1] == pytest.approx(1.375 / math.sqrt(2), rel=1e-14)
        near2, _ = lib.build_riesz(1.9999, 4, 0.5)        # 63-66
        assert near2[0] == pytest.approx(-8.0, rel=1e-3) and near2[1] == pytest.approx(4.0, rel=1e-3)
        assert abs(near2[2]) < 1e-2
        with pytest.raises(ValueError):
            lib.build_riesz(1.0000001, 4, 1.0)            # 74-75
        with pytest.raises(ValueError):
            lib.build_riesz(2.1, 4, 1.0)


def test_toeplitz_matvec_known_answers(ref):
    """test_toeplitz.cpp:78-112"""
    x = np.array([0.5, -2, 3, 7])
    assert np.allclose(ref.toeplitz_matvec([1, 0, 0, 0], [1, 0, 0, 0], x), x, rtol=1e-14)
    assert np.allclose(ref.toeplitz_matvec([2, 1], [2, 3], [1, 1]), [5, 3], rtol=1e-14)
    assert np.allclose(ref.toeplitz_matvec([2, 1], [2, 3], [1, 1], True), [3, 5], rtol=1e-14)
    with pytest.raises(ValueError):
        ref.toeplitz_matvec([2, 1], [2, 3], [1, 2, 3])
    rng = np.random.default_rng(5)
    for n in (1, 2, 3, 8, 17, 64):
        col, row = rng.standard_normal(n), rng.standard_normal(n)
        row[0] = col[0]
        T = dense_toeplitz(col, row)
        x = rng.standard_normal(n)
        s = max(1.0, np.abs(T @ x).max())
        assert np.abs(ref.toeplitz_matvec(col, row, x) - T @ x).max() / s < 1e-12
        assert np.abs(ref.toeplitz_matvec(col, row, x, True) - T.T @ x).max() / s < 1e-12


def test_tchan_and_circulant_eigs(ref, port):
    """test_circulant.cpp:25-89"""
    fc, eig = ref.tchan(*ref.build_caputo(0.5, 3, 1.0))
    assert np.allclose(fc, [1.0, -1 / 3, -0.125 / 3], rtol=1e-14)
    fc2, eig2 = port.tchan(*ref.build_caputo(0.5, 3, 1.0))
    assert np.allclose(fc2, fc, rtol=1e-15) and np.allclose(eig2, eig, rtol=1e-14)
    assert np.allclose(ref.circulant_eigs([0, 1, 0, 0]), [1, -1j, -1, 1j], atol=1e-14)
    a = -0.37
    e = ref.circulant_eigs([a, a, a, a])
    assert abs(e[0] - 4 * a) < 1e-14 and np.abs(e[1:]).max() < 1e-14


def test_preconditioner_known_answers(ref):
    """test_circulant.cpp:117-151: lambda_B == 0 gives lambda_S = rho(1+1/delta);
    identity and halving solves."""
    from oracle.pyoracle import RefPc
    zero = RefPc.from_lam_b(ref, np.zeros(8, dtype=complex), 2, 1.3, 0.7, 1e-4, 1.0)
    assert np.allclose(zero.lam_s(), 1.3 * (1 + 1 / 0.7), rtol=1e-15)
    r = ref.randn(31, 27)
    ident = RefPc.from_lam_b(ref, np.zeros(27, dtype=complex), 3, 0.5, 1.0, 1e-4, 1.0)
    assert np.allclose(ident.solve(r), r, rtol=1e-13, atol=1e-15)
    half = RefPc.from_lam_b(ref, np.zeros(27, dtype=complex), 3, 1.0, 1.0, 1e-4, 1.0)
    assert np.allclose(half.solve(r), r / 2, rtol=1e-13, atol=1e-15)
    with pytest.raises(ValueError):
        half.solve(np.zeros(5))


def test_scaling_known_answer(ref):
    """test_problem.cpp:126-135: psi at n=8 is 9^-1.3"""
    s = ref.scaling(0.7, 1.3, 1.3, 8)
    assert s[0] == pytest.approx(9.0 ** -1.3, rel=1e-14)


# ------------------------------------------- restatement vs the reference
@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_port_matches_reference_default_operator(ref, port, n):
    h = 1.0 / (n + 1)
    rop = ref.op_spec(0.7, 1.3, 1.3, n)
    t, r1, r2 = ref.build_caputo(0.7, n, h), ref.build_riesz(1.3, n, h), ref.build_riesz(1.3, n, h)
    pop = port.op((n, n, n), t, r1, r2, rop.psi)
    x = ref.randn(3 + n, n ** 3)
    for adj in (False, True):
        a = rop.apply(x, adj)
        assert rel(pop.apply(x, adj), a) < 1e-13
        assert rel(pop.apply(x, adj, direct=True), a) < 1e-13  # independent algorithm
    rpc = rop.assemble_precond(1.618, 0.4, 1e-4)
    ppc = pop.assemble_precond(1.618, 0.4, 1e-4)
    assert rel(ppc.solve(x), rpc.solve(x)) < 1e-13


def test_dense_kronecker_unit_basis(ref):
    """oracle.cpp:316-345 check 1 (matvec_unit_basis, 1e-13) restated with numpy."""
    n = 3
    h = 1.0 / (n + 1)
    rop = ref.op_spec(0.7, 1.3, 1.3, n)
    C = dense_toeplitz(*ref.build_caputo(0.7, n, h))
    L1 = dense_toeplitz(*ref.build_riesz(1.3, n, h))
    L2 = dense_toeplitz(*ref.build_riesz(1.3, n, h))
    I = np.eye(n)
    B = rop.psi * (np.kron(C, np.kron(I, I)) - np.kron(I, np.kron(L1, I) + np.kron(I, L2)))
    scale = np.abs(B).max()
    for j in range(n ** 3):
        e = np.zeros(n ** 3)
        e[j] = 1.0
        assert np.abs(rop.apply(e) - B[:, j]).max() / scale < 1e-13


def test_fault_injection_detected(ref):
    """test_oracle.cpp:179-188 analogue: perturbing one coefficient by 1e-6
    must fail the unit-basis check."""
    n = 2
    h = 1.0 / 3
    t, r1, r2 = ref.build_caputo(0.7, n, h), ref.build_riesz(1.3, n, h), ref.build_riesz(1.3, n, h)
    good = ref.op(n, t, r1, r2, 0.1)
    bad_col = r2[0].copy()
    bad_col[1] += 1e-6
    bad = ref.op(n, t, r1, (bad_col, bad_col), 0.1)
    e = np.zeros(8)
    e[1] = 1.0
    assert np.abs(good.apply(e) - bad.apply(e)).max() > 1e-8


# ------------------------------------------------------- golden fixtures
def test_golden_small_reproduces(ref, port, golden):
    """The committed fixtures still come out of the reference (and the port)."""
    for n in (2, 3, 4, 8):
        op = ref.op_spec(0.7, 1.3, 1.3, n)
        x = golden[f"spec{n}_x"]
        assert np.array_equal(op.apply(x, False), golden[f"spec{n}_Bx"])
        assert np.array_equal(op.apply(x, True), golden[f"spec{n}_BTx"])
    for n in (4, 8):
        c = baseline_problem("C0", Shape(n, n, n))
        pop = port.op((n, n, n), c["time"], c["r1"], c["r2"], c["psi"])
        x = golden[f"ie{n}_x"]
        assert rel(pop.apply(x), golden[f"ie{n}_Bx"]) < 1e-14
        assert rel(pop.assemble_precond(1.0, 1.0, c["gamma"]).solve(x), golden[f"ie{n}_Minv_x"]) < 1e-14


def test_golden_c0_summary_present():
    """The full C0 reference solve (tests/golden/ref_c0_solve.*) when generated."""
    import json
    p = os.path.join(HERE, "golden", "ref_c0_solve.json")
    if not os.path.exists(p):
        pytest.skip("C0 golden not generated yet")
    s = json.load(open(p))
    assert s["converged"] and s["admm_iterations"] > 0
    h = np.load(os.path.join(HERE, "golden", "ref_c0_solve.npz"))["history"]
    assert h.shape[0] == s["admm_iterations"] and int(h[:, 5].sum()) == s["total_krylov"]


def test_baseline_mapping():
    """implicit Euler = GL alpha=1 bidiagonal; psi choice."""
    col, row = implicit_euler(4, 0.25)
    assert list(col) == [4.0, -4.0, 0.0, 0.0] and list(row) == [4.0, 0.0, 0.0, 0.0]
    c = baseline_problem("C0")
    assert c["psi"] == pytest.approx(33.0 ** -1.5, rel=1e-15)
    yb = synthetic_ybar("sin", Shape(2, 3, 4))
    assert yb.shape == (24,) and np.isfinite(yb).all()


def test_port_threads_bit_identical(port):
    """The fibre-parallel port (used for the full-size C3/C4 parity tests)
    gives the serial loop's results bit for bit: operator, adjoint,
    preconditioner and a PCG solve."""
    from oracle.pyoracle import PortAdmm
    shape = (6, 20, 24)
    c = baseline_problem("C3", Shape(*shape))
    pop = port.op(shape, c["time"], c["r1"], c["r2"], c["psi"])
    ppc = pop.assemble_precond(1.0, 1.0, c["gamma"])
    x = np.random.default_rng(3).standard_normal(pop.size)
    out = {}
    t0 = port.get_threads()
    try:
        for t in (1, 5):
            port.set_threads(t)
            adm = PortAdmm(port, pop, ppc, c["gamma"], 1.0, 1.0, y_lo=c["y"][0], y_hi=c["y"][1],
                           u_lo=c["u"][0], u_hi=c["u"][1], tol_primal=1e-6, max_inner=400,
                           fixed_tol=1e-8, ybar=x)
            y, r = adm.pcg(adm.build_rhs()[0])
            out[t] = (pop.apply(x), pop.apply(x, True), ppc.solve(x), y, r["iterations"])
    finally:
        port.set_threads(t0)
    for a, b in zip(out[1], out[5]):
        assert np.array_equal(a, b)


def test_numpy_restatement_vs_port(port):
    """oracle/np_fdeopt.py (pocketfft backend, the noise-floor checker) agrees
    with the C restatement: operators 1e-14, PCG counts and residuals of
    three ADMM steps."""
    from oracle.np_fdeopt import NpAdmm, NpOperator, NpPrecond
    from oracle.pyoracle import PortAdmm
    shape = (5, 12, 10)
    c = baseline_problem("C3", Shape(*shape))
    op = NpOperator(shape, c["time"], c["r1"], c["r2"], c["psi"])
    pc = NpPrecond(op, 1.0, 1.0, c["gamma"])
    pop = port.op(shape, c["time"], c["r1"], c["r2"], c["psi"])
    ppc = pop.assemble_precond(1.0, 1.0, c["gamma"])
    x = np.random.default_rng(9).standard_normal(op.size)
    assert rel(op.apply(x), pop.apply(x)) < 1e-14
    assert rel(op.apply(x, True), pop.apply(x, True)) < 1e-14
    assert rel(pc.solve(x), ppc.solve(x)) < 1e-14
    a = NpAdmm(op, pc, c["gamma"], 1.0, 1.0, y_lo=c["y"][0], y_hi=c["y"][1], u_lo=c["u"][0],
               u_hi=c["u"][1], ybar=x)
    b = PortAdmm(port, pop, ppc, c["gamma"], 1.0, 1.0, y_lo=c["y"][0], y_hi=c["y"][1],
                 u_lo=c["u"][0], u_hi=c["u"][1], tol_primal=1e-6, max_inner=400, fixed_tol=1e-8,
                 ybar=x)
    for _ in range(3):
        s1, s2 = a.step(), b.step()
        assert abs(s1["inner_iters"] - s2["inner_iters"]) <= 1
        for k in ("r_eq", "r_u", "dual_inf"):
            assert abs(s1[k] - s2[k]) <= 1e-10 * abs(s2[k])
