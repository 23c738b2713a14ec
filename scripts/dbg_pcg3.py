import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1907_13428_b200 import Context, make_problem
ctx = Context(0)
n = 4
c, op, pc, drv = make_problem("C0", (n, n, n), ctx=ctx)
b, _ = drv.build_rhs()
def rel(a, e): return np.linalg.norm(a - e) / np.linalg.norm(e)
xg, res = drv.pcg(b, tol=1e-8, max_inner=0)
print("r0 vs rhs", rel(drv.debug_get("r"), b), "z0 vs M rhs", rel(drv.debug_get("z"), pc.solve(b)), "p0", rel(drv.debug_get("p"), pc.solve(b)))
sc = drv.debug_get("scalars"); print("scal", sc[:8], "rz expect", b @ pc.solve(b))
