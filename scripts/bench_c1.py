"""BASELINE C1 operator microbenchmark: 2-level Toeplitz matvec and 2-level
T. Chan preconditioner solve on 256 slices of 1023 x 1023 (N = 267,911,424),
fp64, seeded N(0,1) input; device time per call with CUDA events; HBM
fraction against the SURVEY.md 8d pass models (matvec 5N, solve 6N doubles).
Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1907_13428_b200 import Context, make_c1, randn  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ctx = Context(0)
op, pc = make_c1(ctx=ctx)
N = op.size
x = torch.from_numpy(randn(1, N)).cuda()
y = torch.empty_like(x)
st = torch.cuda.ExternalStream(ctx.stream)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]


def timed(fn):
    for _ in range(2):
        fn()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    ctx.synchronize()
    return e0.elapsed_time(e1) / reps


torch.cuda.synchronize()
l0 = ctx.launch_count
t_mv = timed(lambda: op.apply_dev(x, y))
l1 = ctx.launch_count
t_pc = timed(lambda: pc.solve_dev(x, y))
l2 = ctx.launch_count
res = {"config": "C1 256 x (1023, 1023) 2-level Toeplitz matvec + 2-level T. Chan solve", "N": N,
       "matvec_ms": t_mv, "precond_ms": t_pc,
       "matvec_hbm_frac": 5 * 8 * N / (t_mv * 1e-3) / (peak * 1e9),
       "precond_hbm_frac": 6 * 8 * N / (t_pc * 1e-3) / (peak * 1e9),
       "launches_per_matvec": (l1 - l0) / (reps + 2), "launches_per_solve": (l2 - l1) / (reps + 2),
       "peak_gbs": peak}
print(json.dumps(res))
