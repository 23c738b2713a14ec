"""B200-native (sm_100a) hot path of the fractional-diffusion ADMM solver.

Python mirror of the reference's operator / preconditioner / Krylov / ADMM API
(/root/reference/proj/include/fdeopt/{toeplitz,circulant,admm}.hpp) over the
C ABI in include/fdg.h.  All arithmetic runs in lib/libfdg.so on the GPU; the
import fails if the library is missing (no CPU fallback).
"""
from .api import (  # noqa: F401
    Context, ConstraintOperator, CirculantPreconditioner, SpatialPreconditioner,
    assemble_spatial_precond, AdmmConfig, AdmmDriver, IterRecord,
    PcgResult, assemble_precond, solve, frac_coeffs, build_riesz, build_caputo, tchan, randn,
    implicit_euler, FdgError,
)
from .workloads import baseline_config, synthetic_ybar, make_problem, make_c1, c1_factors  # noqa: F401
