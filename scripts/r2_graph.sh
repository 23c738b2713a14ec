timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "graph or pcg_host_x0 or admm_five or apply_S" > gpurun_out/graph_t.log 2>&1; echo t_rc=$?; tail -15 gpurun_out/graph_t.log
for nm in 0 2097152; do
FDG_PCG_GRAPH_NMAX=$nm timeout 300 python - <<'PY'
import time, os, torch
from paper_1907_13428_b200 import Context, make_problem, solve
ctx = Context(0)
c, op, pc, drv = make_problem("C0", ctx=ctx)
t0 = time.perf_counter(); res = solve(drv); t = time.perf_counter() - t0
h = res["history"]
print(f"nmax={os.environ['FDG_PCG_GRAPH_NMAX']} C0 solve {t:.2f} s steps {res['iterations']} krylov {sum(r.inner_iters for r in h)} pcg {sum(r.pcg_ms for r in h)/1e3:.2f} s launches {ctx.launch_count}")
PY
done
