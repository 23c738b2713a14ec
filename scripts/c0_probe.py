"""C0 PCG probe: one zero-state solve (launch list / timing of the latency-bound config)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1907_13428_b200 import Context, make_problem
ctx = Context(0)
c, op, pc, drv = make_problem("C0", ctx=ctx)
rhs, _ = drv.build_rhs()
rd = torch.tensor(rhs, device="cuda")
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    x = torch.zeros_like(rd); torch.cuda.synchronize()
    r = drv.pcg_dev(rd, x, 1e-8, 400)
    print(f"its {r.iterations} ms {r.ms:.3f} us/it {1e3 * r.ms / r.iterations:.1f}")
