"""One PCG solve of a BASELINE config (for ncu captures of the hot kernels).
CONFIG=C2|C3|C4 (real parameters; default C2), SHAPE="nt n1 n2" overrides the
grid, MAXIT caps the Krylov iterations (default 3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1907_13428_b200 import Context, make_problem
name = os.environ.get("CONFIG", "C2")
shape = tuple(int(v) for v in os.environ["SHAPE"].split()) if "SHAPE" in os.environ else None
ctx = Context(0)
c, op, pc, drv = make_problem(name, shape, ctx=ctx)
N = op.size
rhs = torch.empty(N, dtype=torch.float64, device="cuda")
x = torch.zeros_like(rhs)
torch.cuda.synchronize()
drv.build_rhs_dev(rhs)
ctx.synchronize()
r = drv.pcg_dev(rhs, x, 1e-8, int(os.environ.get("MAXIT", "3")))
ctx.synchronize()
print("pcg", r)
