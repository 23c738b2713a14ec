"""One C1 2-level matvec and one 2-level T. Chan solve (256 x 1023^2), for
ncu captures of their kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1907_13428_b200 import Context, make_c1, randn
ctx = Context(0)
op, pc = make_c1(ctx=ctx)
x = torch.from_numpy(randn(1, op.size)).cuda()
y = torch.empty_like(x)
torch.cuda.synchronize()
op.apply_dev(x, y)
pc.solve_dev(x, y)
ctx.synchronize()
print("c1 ok", ctx.launch_count)
