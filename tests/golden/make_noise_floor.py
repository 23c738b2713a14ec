"""Cross-implementation noise floor of the full C0 ADMM solve:
the numpy/pocketfft restatement (oracle/np_fdeopt.py) run to convergence on
the exact C0 inputs of the committed reference solve (ref_c0_solve.*), and
its distance to the reference (FFTW3-shim) solve.  Writes
tests/golden/np_c0_solve.json.  CPU only, ~10 min:

    python tests/golden/make_noise_floor.py
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Shape, baseline_problem  # noqa: E402
from oracle.np_fdeopt import NpAdmm, NpOperator, NpPrecond  # noqa: E402


def main():
    ref = json.load(open(os.path.join(HERE, "ref_c0_solve.json")))
    g = np.load(os.path.join(HERE, "ref_c0_solve.npz"))
    H = g["history"]
    c = baseline_problem("C0", Shape(32, 32, 32))
    op = NpOperator((32, 32, 32), c["time"], c["r1"], c["r2"], c["psi"])
    pc = NpPrecond(op, 1.0, 1.0, c["gamma"])
    adm = NpAdmm(op, pc, c["gamma"], 1.0, 1.0, u_lo=c["u"][0], u_hi=c["u"][1], tol_primal=1e-6,
                 max_inner=400, fixed_tol=1e-8, ybar=g["ybar"])
    t0 = time.time()
    inner = []
    while True:
        r = adm.step()
        inner.append(r["inner_iters"])
        if r["converged"] or len(inner) >= H.shape[0] + 2000:
            break
    secs = time.time() - t0
    inner = np.array(inner)
    n = min(len(inner), H.shape[0])
    d = np.abs(inner[:n] - H[:n, 5])

    def rdiff(a, b):
        return float(abs(a - b) / abs(b)) if b != 0 else float(abs(a - b))

    out = {
        "what": "numpy/pocketfft restatement vs the unchanged reference (FFTW3 shim), C0 full solve",
        "admm_iterations": int(len(inner)), "ref_admm_iterations": ref["admm_iterations"],
        "total_krylov": int(inner.sum()), "ref_total_krylov": ref["total_krylov"],
        "max_abs_dkrylov_per_step": int(d.max()), "steps_with_dkrylov": int((d > 0).sum()),
        "converged": bool(r["converged"]),
        "final": {k: r[k] for k in ("r_eq", "r_y", "r_u", "dual_inf")},
        "objective": adm.objective(),
        "rel_diff_vs_ref": {
            "r_eq": rdiff(r["r_eq"], ref["r_eq"]), "r_u": rdiff(r["r_u"], ref["r_u"]),
            "dual_inf": rdiff(r["dual_inf"], ref["dual_inf"]),
            "objective": rdiff(adm.objective(), ref["objective"]),
            "y": float(np.linalg.norm(adm.y - g["y"]) / np.linalg.norm(g["y"])),
            "v": float(np.linalg.norm(adm.v - g["v"]) / np.linalg.norm(g["v"])),
        },
        "abs_diff_vs_ref": {k: float(abs(r[k] - ref[k])) for k in ("r_eq", "r_y", "r_u", "dual_inf")},
        "seconds": secs,
    }
    with open(os.path.join(HERE, "np_c0_solve.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
