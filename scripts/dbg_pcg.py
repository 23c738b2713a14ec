import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1907_13428_b200 import Context, make_problem
ctx = Context(0)
n = 4
c, op, pc, drv = make_problem("C0", (n, n, n), ctx=ctx)
b, _ = drv.build_rhs()
def rel(a, e): return np.linalg.norm(a - e) / np.linalg.norm(e)
x = np.zeros_like(b); r = b.copy(); z = pc.solve(r); p = z.copy(); rz = r @ z
q = drv.apply_S(p); pq = p @ q; a = rz / pq
x1 = x + a * p; r1 = r - a * q
xg, res = drv.pcg(b, tol=1e-8, max_inner=1)
sc = drv.debug_get("scalars")
print("scalars", sc[:8])
print("expect rz", rz, "pq", pq, "rr", r1 @ r1)
print("r1", rel(drv.debug_get("r"), r1))
z1 = pc.solve(r1)
print("z1", rel(drv.debug_get("z"), z1), "rz1", r1 @ z1)
beta = (r1 @ z1) / rz
print("p1", rel(drv.debug_get("p"), z1 + beta * p), "beta", beta)
print("vp/w/u norms", [np.linalg.norm(drv.debug_get(k)) for k in ("u", "w", "vp")])
rg = drv.debug_get("r")
d = b - rg
aeff = (d @ q) / (q @ q)
print("alpha_eff", aeff, "alpha", a, "resid of fit", np.linalg.norm(d - aeff * q) / np.linalg.norm(d))
qq = d / a
print("q_gpu vs q rel", rel(qq, q))
N = b.size; nt = n; sl = N // nt
for k in range(nt):
    print(" slice", k, rel(qq[k*sl:(k+1)*sl], q[k*sl:(k+1)*sl]))
