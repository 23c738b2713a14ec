"""ctypes binding of include/fdg.h (the product's C ABI).

The library must exist (built by ``paper_1907_13428_b200.build``); there is no
CPU fallback: importing this module without ``lib/libfdg.so`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FDG_LIB") or os.path.join(PKG, "lib", "libfdg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_1907_13428_b200/build.py` "
        "(the B200 path has no CPU fallback)")

lib = C.CDLL(LIB_PATH)

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p

FDG_OK, FDG_EINVAL, FDG_ENUMERIC, FDG_ECUDA, FDG_EUNSUPPORTED, FDG_ENOMEM = range(6)
FIELDS = dict(y=0, v=1, z_y=2, z_v=3, p=4, w_y=5, w_v=6, ybar=7, diag_j=8, diag_j2=9, m2=10,
              a2_inv=11, By=12)


class AdmmDesc(C.Structure):
    _fields_ = [("gamma", C.c_double), ("rho", C.c_double), ("delta", C.c_double),
                ("y_lo", C.c_double), ("y_hi", C.c_double), ("u_lo", C.c_double),
                ("u_hi", C.c_double), ("tol_primal", C.c_double), ("max_outer", C.c_int),
                ("max_inner", C.c_int), ("inner_tol_floor", C.c_double),
                ("inner_tol_factor", C.c_double), ("fixed_krylov_tol", C.c_double),
                ("warm_start", C.c_int)]


class IterRecord(C.Structure):
    _fields_ = [("iter", C.c_int), ("r_eq", C.c_double), ("r_y", C.c_double),
                ("r_u", C.c_double), ("dual_inf", C.c_double), ("inner_iters", C.c_int),
                ("inner_tol", C.c_double), ("converged", C.c_int), ("pcg_converged", C.c_int),
                ("pcg_rel_residual", C.c_double), ("pcg_ms", C.c_double), ("step_ms", C.c_double)]


class PcgResult(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("rel_residual", C.c_double),
                ("ms", C.c_double)]


def _sig(name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


_st = C.c_int
_sig("fdg_last_error", C.c_char_p)
_sig("fdg_last_numeric_code", C.c_int)
_sig("fdg_version", C.c_char_p)
_sig("fdg_ctx_create", _st, C.c_int, _vp, C.POINTER(_vp))
_sig("fdg_ctx_destroy", _st, _vp)
_sig("fdg_ctx_stream", _vp, _vp)
_sig("fdg_ctx_launch_count", C.c_uint64, _vp)
_sig("fdg_ctx_synchronize", _st, _vp)
_sig("fdg_frac_coeffs", _st, C.c_double, C.c_int, _dp)
_sig("fdg_build_riesz", _st, C.c_double, C.c_int, C.c_double, _dp, _dp)
_sig("fdg_build_caputo", _st, C.c_double, C.c_int, C.c_double, _dp, _dp)
_sig("fdg_tchan", _st, C.c_int, _dp, _dp, _dp, _dp)
_sig("fdg_randn", _st, C.c_uint64, C.c_size_t, _dp)
_sig("fdg_op_create", _st, _vp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, C.c_double,
     C.POINTER(_vp))
_sig("fdg_op_destroy", _st, _vp)
_sig("fdg_op_size", C.c_size_t, _vp)
_sig("fdg_op_psi", C.c_double, _vp)
_sig("fdg_op_apply", _st, _vp, _vp, _vp, C.c_int)
_sig("fdg_op_apply_host", _st, _vp, _dp, C.c_size_t, _dp, C.c_size_t, C.c_int)
_sig("fdg_pc_assemble", _st, _vp, C.c_double, C.c_double, C.c_double, C.POINTER(_vp))
_sig("fdg_pc_create", _st, _vp, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, C.c_double, C.c_double,
     C.c_double, C.c_double, C.POINTER(_vp))
_sig("fdg_pc_destroy", _st, _vp)
_sig("fdg_pc_solve", _st, _vp, _vp, _vp)
_sig("fdg_pc_solve_host", _st, _vp, _dp, C.c_size_t, _dp, C.c_size_t)
_sig("fdg_pc_lam_s_host", _st, _vp, _dp)
_sig("fdg_pc2_create", _st, _vp, C.c_int, C.c_int, C.c_int, _dp, _dp, C.POINTER(_vp))
_sig("fdg_pc2_assemble", _st, _vp, C.POINTER(_vp))
_sig("fdg_admm_create", _st, _vp, _vp, C.POINTER(AdmmDesc), _dp, C.POINTER(_vp))
_sig("fdg_admm_destroy", _st, _vp)
_sig("fdg_admm_step", _st, _vp, C.POINTER(IterRecord))
_sig("fdg_admm_converged", C.c_int, _vp)
_sig("fdg_admm_stagnations", C.c_int, _vp)
_sig("fdg_admm_get", _st, _vp, C.c_int, _dp)
_sig("fdg_admm_set", _st, _vp, C.c_int, _dp)
_sig("fdg_admm_field_ptr", _st, _vp, C.c_int, C.POINTER(_vp))
_sig("fdg_admm_apply_S", _st, _vp, _vp, _vp)
_sig("fdg_admm_build_rhs", _st, _vp, _vp, _vp)
_sig("fdg_admm_pcg", _st, _vp, _vp, _vp, C.c_double, C.c_int, C.POINTER(PcgResult))
_sig("fdg_admm_pcg_host", _st, _vp, _dp, _dp, C.c_double, C.c_int, C.POINTER(PcgResult))
_sig("fdg_admm_dual_inf", _st, _vp, _dp)
_sig("fdg_admm_objective", _st, _vp, _dp)
_sig("fdg_admm_profile_passes", _st, _vp, C.c_int, _dp, _dp)
_sig("fdg_set_pcg_graph_nmax", _st, C.c_longlong, C.POINTER(C.c_longlong))
_sig("fdg_admm_debug_get", _st, _vp, C.c_int, _dp)

PASS_NAMES = ["K1_row_p_update_B", "K2_col_S_mid", "K3_row_BT_update", "P1_hartley_x2",
              "P2_hartley_x1", "P3_t_filter", "P4_hartley_x1", "P5_hartley_x2_dot", "X_axpy"]


class FdgError(RuntimeError):
    def __init__(self, code, msg, numeric=0):
        super().__init__(msg)
        self.code, self.numeric = code, numeric


def check(rc: int) -> None:
    if rc == FDG_OK:
        return
    msg = lib.fdg_last_error().decode()
    if rc == FDG_EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise FdgError(rc, msg, lib.fdg_last_numeric_code())
