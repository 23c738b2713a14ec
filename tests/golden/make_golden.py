"""Generate the committed golden fixtures from the UNCHANGED reference.

Run in the build container (it needs oracle/_ref, built from /root/reference):

    python tests/golden/make_golden.py small   # seconds: operator/precond/PCG/ADMM vectors
    python tests/golden/make_golden.py c0      # ~20 min: the full BASELINE C0 solve history

Inputs follow SURVEY.md §8(d): std::mt19937_64(seed) + std::normal_distribution
(libstdc++), drawn in layout order; the desired state of C0 is
sin(pi x1) sin(pi x2) e^t + 0.01 xi with seed 1.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Shape, baseline_problem, ref_lib, synthetic_ybar  # noqa: E402
from oracle.pyoracle import RefAdmm  # noqa: E402


def small():
    R = ref_lib()
    out = {}
    # Reference-default operator (Caputo alpha, Riesz betas), cube sizes.
    for n in (2, 3, 4, 8, 16):
        op = R.op_spec(0.7, 1.3, 1.3, n)
        x = R.randn(100 + n, n ** 3)
        out[f"spec{n}_x"] = x
        out[f"spec{n}_Bx"] = op.apply(x, False)
        out[f"spec{n}_BTx"] = op.apply(x, True)
        pc = op.assemble_precond(1.618, 0.4, 1e-4)
        out[f"spec{n}_Minv_x"] = pc.solve(x)
    # BASELINE (implicit Euler) operator at cube sizes.
    for n in (4, 8, 16):
        c = baseline_problem("C0", Shape(n, n, n))
        op = R.op(n, c["time"], c["r1"], c["r2"], c["psi"])
        pc = op.assemble_precond(1.0, 1.0, c["gamma"])
        x = R.randn(200 + n, n ** 3)
        out[f"ie{n}_x"] = x
        out[f"ie{n}_Bx"] = op.apply(x, False)
        out[f"ie{n}_BTx"] = op.apply(x, True)
        out[f"ie{n}_Minv_x"] = pc.solve(x)
        ybar = synthetic_ybar("sin", Shape(n, n, n))
        adm = RefAdmm(R, op, pc, c["gamma"], 1.0, 1.0, u_lo=c["u"][0], u_hi=c["u"][1],
                      tol_primal=1e-6, max_inner=400, fixed_tol=1e-8, ybar=ybar)
        out[f"ie{n}_ybar"] = ybar
        out[f"ie{n}_Sx"] = adm.apply_S(x)
        rhs, _ = adm.build_rhs()
        y, res = adm.pcg(rhs, tol=1e-8, max_inner=400)
        out[f"ie{n}_rhs0"] = rhs
        out[f"ie{n}_pcg0_y"] = y
        out[f"ie{n}_pcg0_iters"] = np.array([res["iterations"]])
        recs = [adm.step() for _ in range(5)]
        out[f"ie{n}_steps_inner"] = np.array([r["inner_iters"] for r in recs])
        out[f"ie{n}_steps_res"] = np.array([[r["r_eq"], r["r_y"], r["r_u"], r["dual_inf"]]
                                            for r in recs])
        for f in ("y", "v", "z_v", "p", "w_v"):
            out[f"ie{n}_after5_{f}"] = adm.get(f)
        out[f"ie{n}_after5_obj"] = np.array([adm.objective()])
    np.savez_compressed(os.path.join(HERE, "ref_small.npz"), **out)
    print("wrote ref_small.npz", len(out), "arrays")


def c0():
    R = ref_lib()
    c = baseline_problem("C0")
    s = c["shape"]
    n = s.nt
    ybar = synthetic_ybar("sin", s)
    op = R.op(n, c["time"], c["r1"], c["r2"], c["psi"])
    pc = op.assemble_precond(c["rho"], c["delta"], c["gamma"])
    adm = RefAdmm(R, op, pc, c["gamma"], c["rho"], c["delta"], u_lo=c["u"][0], u_hi=c["u"][1],
                  tol_primal=c["tol_primal"], max_outer=100000, max_inner=c["max_inner"],
                  fixed_tol=c["krylov_tol"], ybar=ybar)
    hist = []
    t0 = time.time()
    pcg_s = 0.0
    while True:
        r = adm.step()
        pcg_s += r["pcg_seconds"]
        hist.append([r["iter"], r["r_eq"], r["r_y"], r["r_u"], r["dual_inf"], r["inner_iters"]])
        if r["converged"] or r["iter"] >= 100000:
            break
    wall = time.time() - t0
    H = np.array(hist)
    np.savez_compressed(os.path.join(HERE, "ref_c0_solve.npz"), history=H, ybar=ybar,
                        y=adm.get("y"), v=adm.get("v"), p=adm.get("p"))
    summary = dict(config="C0", shape=[n, n, n], admm_iterations=int(H[-1, 0]),
                   converged=bool(r["converged"]), total_krylov=int(H[:, 5].sum()),
                   objective=adm.objective(), r_eq=r["r_eq"], r_y=r["r_y"], r_u=r["r_u"],
                   dual_inf=r["dual_inf"], wall_seconds=wall, pcg_seconds=pcg_s,
                   krylov_per_s=float(H[:, 5].sum() / pcg_s), threads=1,
                   note="unchanged reference sources + FFTW3 shim (oracle/shim), g++ -O3")
    with open(os.path.join(HERE, "ref_c0_solve.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    {"small": small, "c0": c0}[sys.argv[1]]()
