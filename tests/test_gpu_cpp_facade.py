"""The C++ façade (include/fdeopt_b200.hpp) drives the GPU path like a
reference user would; its first 5 ADMM steps match the unchanged reference."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_facade_matches_reference(tmp_path, ref):
    from oracle import Shape, baseline_problem
    from oracle.pyoracle import RefAdmm
    lib = os.path.join(ROOT, "paper_1907_13428_b200", "lib")
    exe = tmp_path / "facade_c0"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_c0.cpp"), "-L", lib, "-lfdg",
                    f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    steps = [l.split() for l in out.splitlines() if l.startswith("step")]
    assert "size check ok" in out and len(steps) == 5
    n = 8
    c = baseline_problem("C0", Shape(n, n, n))
    rng_y = ref.randn(1, n ** 3)
    t = (np.arange(n) + 1.0) / n
    x = (np.arange(n) + 1.0) / (n + 1)
    T, X1, X2 = np.meshgrid(t, x, x, indexing="ij")
    ybar = (np.sin(np.pi * X1) * np.sin(np.pi * X2) * np.exp(T)).ravel() + 0.01 * rng_y
    rop = ref.op(n, c["time"], c["r1"], c["r2"], c["psi"])
    rpc = rop.assemble_precond(1.0, 1.0, c["gamma"])
    adm = RefAdmm(ref, rop, rpc, c["gamma"], 1.0, 1.0, u_lo=-2.0, u_hi=1.5, tol_primal=1e-6,
                  max_inner=400, fixed_tol=1e-8, ybar=ybar)
    for s in steps:
        r = adm.step()
        assert abs(int(s[3]) - r["inner_iters"]) <= 1
        assert abs(float(s[5]) - r["r_eq"]) <= 1e-8 * max(abs(r["r_eq"]), 1e-12)
