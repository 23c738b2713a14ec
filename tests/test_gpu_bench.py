"""bench.py keeps the driver's JSON contract (one line; metric/value/unit,
timing rules, roofline, e2e, clocks, launches) -- run small on the GPU."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline", "--admm-steps", "1", "--profile-reps", "2",
                          "--shape", "32", "128", "128", "--configs", "C0"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks", "roofline",
              "iteration_roofline", "steady_state_iteration"):
        assert k in d, k
    assert d["metric"] == "krylov_iters_per_s" and d["unit"] == "it/s" and d["higher_is_better"] is True
    assert d["steps"] == 3 and d["warmup"] >= 3 and d["n_gpus"] == 1 and d["dtype"] == "f64"
    assert d["value"] > 0 and d["gpu_launches"] > 0 and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "it/s" and e["h2d_bytes_per_step"] == 2 * 8 * 32 * 128 * 128
    assert e["d2h_bytes_per_step"] == 8 * 32 * 128 * 128
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["steady_state_iteration"]["ms_per_iteration"] > 0
    # the C0 full ADMM solve: the reference's step and Krylov counts
    c0 = d["admm_solve"]["C0"]
    assert c0["status"] == "converged" and c0["same_counts"], c0
    assert r["traffic"] is None  # no ncu capture for this shape
