import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1907_13428_b200 import Context, make_problem
ctx = Context(0)
n = 4
c, op, pc, drv = make_problem("C0", (n, n, n), ctx=ctx)
b, _ = drv.build_rhs()
z0 = pc.solve(b)
print("b[:3]", b[:3], "z0[:3]", z0[:3], flush=True)
q = drv.apply_S(z0)
print("host q[:3]", q[:3], flush=True)
xg, res = drv.pcg(b, tol=1e-8, max_inner=1)
ctx.synchronize()
print(res, flush=True)
