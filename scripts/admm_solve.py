"""Full ADMM solve of a BASELINE config on the B200 path (the BASELINE
metric's 'ADMM solve time'): fdeopt::solve's outer loop (api.solve) from a
zero state with the fixed Krylov tolerance 1e-8 and tol_primal 1e-6.

    python scripts/admm_solve.py [C2] [max_outer]   -> one JSON line
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1907_13428_b200 import Context, make_problem, solve  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
max_outer = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
ctx = Context(0)
t0 = time.perf_counter()
c, op, pc, drv = make_problem(name, ctx=ctx)
drv.cfg.max_outer = max_outer
torch.cuda.synchronize()
t_setup = time.perf_counter() - t0
last = {}


LOG = os.environ.get("ADMM_LOG")


def cb(rec):
    last["rec"] = rec
    if LOG and rec.iter % 250 == 0:
        with open(LOG, "a") as fh:
            fh.write(f"{rec.iter} {time.perf_counter() - t1:.1f}s r_eq={rec.r_eq:.3e} r_y={rec.r_y:.3e} "
                     f"r_u={rec.r_u:.3e} inner={rec.inner_iters}\n")


t1 = time.perf_counter()
res = solve(drv, cb)
t_solve = time.perf_counter() - t1
rec = last["rec"]
hist = res["history"]
out = {"config": name, "shape": list(c["shape"]), "status": res["status"], "admm_steps": res["iterations"],
       "krylov_total": int(sum(h.inner_iters for h in hist)), "pcg_avg": res["pcg_avg"],
       "solve_seconds": t_solve, "setup_seconds": t_setup,
       "pcg_seconds": sum(h.pcg_ms for h in hist) / 1e3, "step_ms_mean": 1e3 * t_solve / max(1, len(hist)),
       "r_eq": rec.r_eq, "r_y": rec.r_y, "r_u": rec.r_u, "dual_inf": res["dual_inf"], "objective": res["objective"]}
print(json.dumps(out), flush=True)
