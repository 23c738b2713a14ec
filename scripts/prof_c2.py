"""One C2 PCG solve (for ncu captures of the hot kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1907_13428_b200 import Context, make_problem
shape = tuple(int(v) for v in os.environ.get("SHAPE", "256 256 256").split())
ctx = Context(0)
c, op, pc, drv = make_problem("C2", shape, ctx=ctx)
N = op.size
rhs = torch.empty(N, dtype=torch.float64, device="cuda")
x = torch.zeros_like(rhs)
torch.cuda.synchronize()
drv.build_rhs_dev(rhs)
ctx.synchronize()
r = drv.pcg_dev(rhs, x, 1e-8, int(os.environ.get("MAXIT", "3")))
ctx.synchronize()
print("pcg", r)
