"""oracle/ — TEST INFRASTRUCTURE ONLY.

The CPU checker for the B200 path.  Two layers, both loaded through ctypes:

* ``ref``  : ``oracle/_ref/libfdeopt_ref.so`` — the UNCHANGED reference sources
  (/root/reference/proj/src/{fft,problem,toeplitz,circulant,admm}.cpp) built by
  ``oracle/Makefile`` against the FFTW3 shim, plus ``ref_adapter.cpp``.
* ``port`` : ``oracle/build/liboracle.so`` — the plain-C restatement generalized
  to (n_t, n_x1, n_x2) shapes (``fdeopt_oracle.c``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline — never as the product path.
"""
from .pyoracle import (  # noqa: F401
    RefLib, PortLib, ref_lib, port_lib, build_oracle, ORACLE_DIR,
    Shape, implicit_euler, riesz, baseline_problem, randn, synthetic_ybar,
)
