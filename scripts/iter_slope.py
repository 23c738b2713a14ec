"""Per-iteration cost of the device PCG in the launch chain: solve times at
several iteration caps (tol unreachable) -> least-squares slope and
intercept (fixed per-solve cost).  C2 shape unless given."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_13428_b200 import Context, make_problem  # noqa: E402

shape = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) >= 4 else (256, 256, 256)
N = shape[0] * shape[1] * shape[2]
ctx = Context(0)
c, op, pc, drv = make_problem("C2", shape, ctx=ctx, seed=1)
drv.step()
rhs = torch.empty(N, dtype=torch.float64, device="cuda")
x = torch.empty_like(rhs)
torch.cuda.synchronize()
drv.build_rhs_dev(rhs)
ctx.synchronize()
caps = [1, 2, 4, 6, 8, 10, 12]
res = {}
for rep in range(4):
    for k in caps:
        x.zero_()
        torch.cuda.synchronize()
        r = drv.pcg_dev(rhs, x, 1e-30, k)
        if rep:
            res.setdefault(k, []).append(r.ms)
ks = np.array(caps, float)
ts = np.array([np.median(res[k]) for k in caps])
A = np.vstack([ks, np.ones_like(ks)]).T
slope, icpt = np.linalg.lstsq(A, ts, rcond=None)[0]
print("caps", caps)
print("ms", [round(t, 3) for t in ts])
print(f"slope {slope*1e3:.1f} us/iteration  intercept {icpt*1e3:.1f} us")
# converged solve for reference
x.zero_()
torch.cuda.synchronize()
r = drv.pcg_dev(rhs, x, 1e-8, 400)
print(f"tol 1e-8: {r.iterations} its {r.ms:.3f} ms")
