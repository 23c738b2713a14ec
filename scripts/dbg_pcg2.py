import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1907_13428_b200 import Context, make_problem
ctx = Context(0)
n = 4
c, op, pc, drv = make_problem("C0", (n, n, n), ctx=ctx)
b, _ = drv.build_rhs()
def rel(a, e): return np.linalg.norm(a - e) / np.linalg.norm(e)
xg, res = drv.pcg(b, tol=1e-8, max_inner=1)
d0 = drv.debug_get("p"); r0 = drv.debug_get("r")
drv.profile_passes(1)
r2 = drv.debug_get("r")
qk = (r0 - r2) / 2.0
qs = drv.apply_S(d0)
print("K3-path q vs apply_S q:", rel(qk, qs))
u = drv.debug_get("u"); w = drv.debug_get("w"); vp = drv.debug_get("vp")
print("norms", np.linalg.norm(qk), np.linalg.norm(qs))
