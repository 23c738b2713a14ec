"""Per-pass device times of the PCG iteration (no solve; works for
timing-only experimental builds).  Usage: FDG_LIB=... [SHAPE="nt n1 n2"] python scripts/pass_times.py [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1907_13428_b200 import Context, make_problem
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
shape = tuple(int(v) for v in os.environ.get("SHAPE", "256 256 256").split())
ctx = Context(0)
c, op, pc, drv = make_problem("C2", shape, ctx=ctx)
p = drv.profile_passes(reps)
print(" ".join(f"{k.split('_')[0]}={v['ms']*1e3:.0f}" for k, v in p.items()))
