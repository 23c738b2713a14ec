"""The drop-in boundary on a GPU-less host: the C-ABI library loads, exports
every entry point include/fdg.h declares, and its host-side setup arithmetic
(coefficients, T. Chan eigenvalues, RNG) is bit-identical to the reference.
No device compute is called here."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "fdg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fdg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header():
    from paper_1907_13428_b200._native import LIB_PATH
    lib = ctypes.CDLL(LIB_PATH)
    names = header_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_1907_13428_b200._native import LIB_PATH
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_setup_bit_identical(ref):
    import paper_1907_13428_b200 as p
    for order in (0.3, 0.7, 1.2, 1.5, 1.8):
        assert np.array_equal(p.frac_coeffs(order, 64), ref.frac_coeffs(order, 64))
    for beta, n, h in [(1.5, 256, 1 / 257), (1.2, 512, 1 / 513), (1.8, 1023, 1 / 1024), (1.3, 1, 1.0)]:
        assert np.array_equal(p.build_riesz(beta, n, h)[0], ref.build_riesz(beta, n, h)[0])
    for alpha, n, h in [(0.5, 3, 1.0), (0.7, 64, 1 / 65)]:
        a, b = p.build_caputo(alpha, n, h), ref.build_caputo(alpha, n, h)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(p.randn(1, 5000), ref.randn(1, 5000))
    for col, row in [ref.build_caputo(0.7, 64, 1 / 65), ref.build_riesz(1.5, 33, 1 / 34)]:
        fc, eig = p.tchan(col, row)
        fc2, eig2 = ref.tchan(col, row)
        assert np.array_equal(fc, fc2)
        assert np.abs(eig - eig2).max() <= 1e-13 * np.abs(eig2).max()


def test_setup_errors_match_reference():
    import paper_1907_13428_b200 as p
    with pytest.raises(ValueError):
        p.build_riesz(1.0000001, 4, 1.0)
    with pytest.raises(ValueError):
        p.build_caputo(1.5, 3, 1.0)
    with pytest.raises(ValueError):
        p.frac_coeffs(2.5, 4)


def test_workload_mapping_matches_oracle():
    from oracle import Shape, baseline_problem
    from paper_1907_13428_b200 import baseline_config
    for name, shape in [("C0", (4, 8, 16)), ("C3", (4, 16, 32)), ("C2", (8, 8, 8))]:
        a = baseline_config(name, shape)
        b = baseline_problem(name, Shape(*shape))
        assert a["psi"] == b["psi"]
        for k_a, k_b in (("time", "time"), ("x1", "r1"), ("x2", "r2")):
            assert np.array_equal(a[k_a][0], b[k_b][0]) and np.array_equal(a[k_a][1], b[k_b][1])


def test_no_cpu_fallback_when_library_missing(tmp_path):
    """Importing the product without its .so fails loudly."""
    import subprocess
    import sys
    code = ("import os; os.environ['FDG_LIB']=%r; import sys; sys.path.insert(0, %r); "
            "import paper_1907_13428_b200") % (str(tmp_path / "missing.so"), ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert r.returncode != 0 and "no CPU fallback" in r.stderr
