"""ctypes bindings for the CPU oracle (TEST INFRASTRUCTURE ONLY; see __init__)."""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

ORACLE_DIR = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libfdeopt_ref.so")
PORT_SO = os.path.join(ORACLE_DIR, "build", "liboracle.so")

_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def build_oracle(ref: bool = True) -> None:
    """Build build/liboracle.so, and oracle/_ref when /root/reference exists."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, *targets], check=True)


class OracleError(RuntimeError):
    pass


class _Lib:
    so_path = ""
    err_fn = ""

    def __init__(self):
        if not os.path.exists(self.so_path):
            raise FileNotFoundError(f"{self.so_path} missing: run `make -C oracle`")
        self.lib = C.CDLL(self.so_path)
        getattr(self.lib, self.err_fn).restype = C.c_char_p

    def check(self, rc: int):
        if rc != 0:
            msg = getattr(self.lib, self.err_fn)().decode()
            if rc == -1:
                raise ValueError(msg)
            raise OracleError(msg)


# --------------------------------------------------------------------------
# The unchanged reference (oracle/_ref)
# --------------------------------------------------------------------------
class RefLib(_Lib):
    so_path = REF_SO
    err_fn = "ref_last_error"

    def __init__(self):
        super().__init__()
        L = self.lib
        for name in ("ref_op_create", "ref_op_create_spec", "ref_op_create_zero",
                     "ref_pc_assemble", "ref_pc_create", "ref_admm_create"):
            getattr(L, name).restype = C.c_void_p
        L.ref_op_create.argtypes = [C.c_int] + [_dp] * 6 + [C.c_double]
        L.ref_op_create_spec.argtypes = [C.c_double] * 3 + [C.c_int]
        L.ref_op_create_zero.argtypes = [C.c_int]
        L.ref_op_destroy.argtypes = [C.c_void_p]
        L.ref_op_psi.argtypes = [C.c_void_p]
        L.ref_op_psi.restype = C.c_double
        L.ref_op_apply.argtypes = [C.c_void_p, _dp, _dp, C.c_long, C.c_long, C.c_int]
        L.ref_pc_assemble.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double]
        L.ref_pc_create.argtypes = [_dp, C.c_int] + [C.c_double] * 4
        L.ref_pc_destroy.argtypes = [C.c_void_p]
        L.ref_pc_solve.argtypes = [C.c_void_p, _dp, _dp, C.c_long, C.c_long]
        L.ref_pc_lam_s.argtypes = [C.c_void_p, _dp]
        L.ref_pc_lam_b.argtypes = [C.c_void_p, _dp]
        L.ref_admm_create.argtypes = ([C.c_void_p, C.c_void_p] + [C.c_double] * 8
                                      + [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                         C.c_int, _dp])
        L.ref_admm_destroy.argtypes = [C.c_void_p]
        L.ref_admm_size.argtypes = [C.c_void_p]
        L.ref_admm_size.restype = C.c_long
        L.ref_admm_psi.argtypes = [C.c_void_p]
        L.ref_admm_psi.restype = C.c_double
        for name in ("ref_admm_get", "ref_admm_set"):
            getattr(L, name).argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_admm_apply_S.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_admm_build_rhs.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_admm_pcg.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int, _dp]
        L.ref_admm_step.argtypes = [C.c_void_p, _dp]
        L.ref_admm_krylov_init.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp]
        L.ref_admm_krylov_iteration.argtypes = [C.c_void_p] + [_dp] * 7
        L.ref_admm_dual_inf.argtypes = [C.c_void_p, _dp]
        L.ref_admm_objective.argtypes = [C.c_void_p, _dp]
        L.ref_randn.argtypes = [C.c_uint64, C.c_long, _dp]
        L.ref_frac_coeffs.argtypes = [C.c_double, C.c_int, _dp]
        L.ref_scaling.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, _dp]
        L.ref_desired_state.argtypes = [C.c_int, _dp]
        L.ref_build_caputo.argtypes = [C.c_double, C.c_int, C.c_double, _dp, _dp]
        L.ref_build_riesz.argtypes = [C.c_double, C.c_int, C.c_double, _dp, _dp]
        L.ref_toeplitz_matvec.argtypes = [C.c_int, _dp, _dp, _dp, _dp, C.c_int]
        L.ref_embed_symbol.argtypes = [C.c_int, _dp, _dp, C.c_int, _dp]
        L.ref_tchan.argtypes = [C.c_int, _dp, _dp, _dp, _dp]
        L.ref_circulant_eigs.argtypes = [C.c_int, _dp, _dp]
        L.ref_dft.argtypes = [C.c_int, _dp, _dp, C.c_int]
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_solve.argtypes = ([C.c_double] * 4 + [C.c_int] + [C.c_double] * 7
                                + [C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int,
                                   C.POINTER(C.c_int), _dp, _dp])

    # ---- 1-D building blocks
    def frac_coeffs(self, order, count):
        out = np.zeros(count)
        self.check(self.lib.ref_frac_coeffs(order, count, _ptr(out)))
        return out

    def scaling(self, alpha, beta1, beta2, n):
        out = np.zeros(4)
        self.check(self.lib.ref_scaling(alpha, beta1, beta2, n, _ptr(out)))
        return out

    def desired_state(self, n):
        out = np.zeros(n ** 3)
        self.check(self.lib.ref_desired_state(n, _ptr(out)))
        return out

    def build_caputo(self, alpha, n, h):
        col, row = np.zeros(n), np.zeros(n)
        self.check(self.lib.ref_build_caputo(alpha, n, h, _ptr(col), _ptr(row)))
        return col, row

    def build_riesz(self, beta, n, h):
        col, row = np.zeros(n), np.zeros(n)
        self.check(self.lib.ref_build_riesz(beta, n, h, _ptr(col), _ptr(row)))
        return col, row

    def toeplitz_matvec(self, col, row, x, transpose=False):
        col, row, x = (np.ascontiguousarray(v, dtype=np.float64) for v in (col, row, x))
        out = np.zeros(len(col))
        if len(x) != len(col):  # toeplitz.cpp:66-67 throws invalid_argument
            raise ValueError("toeplitz_matvec: dimension mismatch")
        self.check(self.lib.ref_toeplitz_matvec(len(col), _ptr(col), _ptr(row), _ptr(x),
                                                _ptr(out), int(transpose)))
        return out

    def embed_symbol(self, col, row, transpose=False):
        n = len(col)
        col, row = (np.ascontiguousarray(v, dtype=np.float64) for v in (col, row))
        out = np.zeros(2 * (n + 1))
        self.check(self.lib.ref_embed_symbol(n, _ptr(col), _ptr(row), int(transpose), _ptr(out)))
        return out[0::2] + 1j * out[1::2]

    def tchan(self, col, row):
        n = len(col)
        col, row = (np.ascontiguousarray(v, dtype=np.float64) for v in (col, row))
        fc, eig = np.zeros(n), np.zeros(2 * n)
        self.check(self.lib.ref_tchan(n, _ptr(col), _ptr(row), _ptr(fc), _ptr(eig)))
        return fc, eig[0::2] + 1j * eig[1::2]

    def circulant_eigs(self, first_col):
        n = len(first_col)
        fc = np.ascontiguousarray(first_col, dtype=np.float64)
        eig = np.zeros(2 * n)
        self.check(self.lib.ref_circulant_eigs(n, _ptr(fc), _ptr(eig)))
        return eig[0::2] + 1j * eig[1::2]

    def dft(self, x, inverse=False):
        x = np.asarray(x, dtype=np.complex128)
        inp = np.ascontiguousarray(np.stack([x.real, x.imag], -1).ravel())
        out = np.zeros_like(inp)
        self.check(self.lib.ref_dft(len(x), _ptr(inp), _ptr(out), int(inverse)))
        return out[0::2] + 1j * out[1::2]

    def randn(self, seed, count):
        out = np.zeros(count)
        self.check(self.lib.ref_randn(seed, count, _ptr(out)))
        return out

    def set_threads(self, t):
        self.lib.ref_set_threads(int(t))

    # ---- handles
    def op(self, n, time, r1, r2, psi):
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (*time, *r1, *r2)]
        h = self.lib.ref_op_create(n, *[_ptr(a) for a in arrs], psi)
        if not h:
            self.check(-1)
        return RefOp(self, h, n)

    def op_spec(self, alpha, beta1, beta2, n):
        h = self.lib.ref_op_create_spec(alpha, beta1, beta2, n)
        if not h:
            self.check(-1)
        return RefOp(self, h, n)

    def op_zero(self, n):
        return RefOp(self, self.lib.ref_op_create_zero(n), n)

    def solve(self, alpha=0.7, beta1=1.3, beta2=1.3, gamma=1e-4, n=8, y_lo=-math.inf,
              y_hi=math.inf, u_lo=-math.inf, u_hi=math.inf, delta=0.4, rho=1.618,
              tol_primal=1e-4, max_outer=500, max_inner=400, warm_start=False):
        summary = np.zeros(6)
        hist = np.zeros(7 * max_outer)
        nh = C.c_int(0)
        y, u = np.zeros(n ** 3), np.zeros(n ** 3)
        self.check(self.lib.ref_solve(alpha, beta1, beta2, gamma, n, y_lo, y_hi, u_lo, u_hi,
                                      delta, rho, tol_primal, max_outer, max_inner,
                                      int(warm_start), _ptr(summary), _ptr(hist), max_outer,
                                      C.byref(nh), _ptr(y), _ptr(u)))
        return dict(status="converged" if summary[0] == 0 else "itercap",
                    iterations=int(summary[1]), pcg_avg=summary[2], misfit=summary[3],
                    dual_inf=summary[4], wall_seconds=summary[5],
                    history=hist[: 7 * nh.value].reshape(-1, 7), y=y, u=u)


class RefOp:
    def __init__(self, lib: RefLib, h, n):
        self.L, self.h, self.n = lib, h, n
        self.size = n ** 3

    def __del__(self):
        if getattr(self, "h", None):
            self.L.lib.ref_op_destroy(self.h)
            self.h = None

    @property
    def psi(self):
        return self.L.lib.ref_op_psi(self.h)

    def apply(self, x, adjoint=False, out_size=None):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(self.size if out_size is None else out_size)
        self.L.check(self.L.lib.ref_op_apply(self.h, _ptr(x), _ptr(out), x.size, out.size,
                                             int(adjoint)))
        return out

    def assemble_precond(self, rho, delta, gamma):
        h = self.L.lib.ref_pc_assemble(self.h, rho, delta, gamma)
        if not h:
            self.L.check(-1)
        return RefPc(self.L, h, self.size, keep=self)


class RefPc:
    def __init__(self, lib, h, size, keep=None):
        self.L, self.h, self.size, self._keep = lib, h, size, keep

    @classmethod
    def from_lam_b(cls, lib: RefLib, lam_b, n, rho, delta, gamma, psi):
        lb = np.ascontiguousarray(np.stack([np.real(lam_b), np.imag(lam_b)], -1).ravel())
        h = lib.lib.ref_pc_create(_ptr(lb), n, rho, delta, gamma, psi)
        if not h:
            lib.check(-1)
        return cls(lib, h, n ** 3)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.lib.ref_pc_destroy(self.h)
            self.h = None

    def solve(self, r, out_size=None):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(self.size if out_size is None else out_size)
        self.L.check(self.L.lib.ref_pc_solve(self.h, _ptr(r), _ptr(z), r.size, z.size))
        return z

    def lam_s(self):
        out = np.zeros(self.size)
        self.L.check(self.L.lib.ref_pc_lam_s(self.h, _ptr(out)))
        return out

    def lam_b(self):
        out = np.zeros(2 * self.size)
        self.L.check(self.L.lib.ref_pc_lam_b(self.h, _ptr(out)))
        return out[0::2] + 1j * out[1::2]


FIELDS = dict(y=0, v=1, z_y=2, z_v=3, p=4, w_y=5, w_v=6, ybar=7, diag_j=8, diag_j2=9, m2=10,
              a2_inv=11, By=12)


class _AdmmBase:
    pfx = ""

    def get(self, name):
        out = np.zeros(self.N)
        self.L.check(getattr(self.L.lib, self.pfx + "admm_get")(self.h, FIELDS[name], _ptr(out)))
        return out

    def set(self, name, val):
        val = np.ascontiguousarray(val, dtype=np.float64)
        assert val.size == self.N
        self.L.check(getattr(self.L.lib, self.pfx + "admm_set")(self.h, FIELDS[name], _ptr(val)))

    def apply_S(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(self.N)
        self.L.check(getattr(self.L.lib, self.pfx + "admm_apply_S")(self.h, _ptr(x), _ptr(out)))
        return out

    def build_rhs(self):
        rhs, r = np.zeros(self.N), np.zeros(self.N)
        self.L.check(getattr(self.L.lib, self.pfx + "admm_build_rhs")(self.h, _ptr(rhs), _ptr(r)))
        return rhs, r

    def pcg(self, rhs, x=None, tol=1e-8, max_inner=400):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.zeros(self.N) if x is None else np.ascontiguousarray(x, dtype=np.float64).copy()
        res = np.zeros(4)
        self.L.check(getattr(self.L.lib, self.pfx + "admm_pcg")(self.h, _ptr(rhs), _ptr(x), tol,
                                                                 max_inner, _ptr(res)))
        return x, dict(iterations=int(res[0]), converged=bool(res[1]), rel_residual=res[2],
                       seconds=res[3])

    def step(self):
        rec = np.zeros(12)
        self.L.check(getattr(self.L.lib, self.pfx + "admm_step")(self.h, _ptr(rec)))
        return dict(iter=int(rec[0]), r_eq=rec[1], r_y=rec[2], r_u=rec[3], dual_inf=rec[4],
                    inner_iters=int(rec[5]), inner_tol=rec[6], converged=bool(rec[7]),
                    pcg_seconds=rec[8], step_seconds=rec[9])

    def dual_inf(self):
        out = np.zeros(1)
        self.L.check(getattr(self.L.lib, self.pfx + "admm_dual_inf")(self.h, _ptr(out)))
        return out[0]

    def objective(self):
        out = np.zeros(1)
        self.L.check(getattr(self.L.lib, self.pfx + "admm_objective")(self.h, _ptr(out)))
        return out[0]


class RefAdmm(_AdmmBase):
    pfx = "ref_"

    def __init__(self, lib: RefLib, op: RefOp, pc: RefPc, gamma, rho, delta, y_lo=-math.inf,
                 y_hi=math.inf, u_lo=-math.inf, u_hi=math.inf, tol_primal=1e-4, max_outer=500,
                 max_inner=400, inner_tol_floor=1e-4, inner_tol_factor=0.05, fixed_tol=0.0,
                 warm_start=False, ybar=None):
        self.L, self._keep = lib, (op, pc)
        yb = None if ybar is None else np.ascontiguousarray(ybar, dtype=np.float64)
        self.h = lib.lib.ref_admm_create(op.h, pc.h, gamma, rho, delta, y_lo, y_hi, u_lo, u_hi,
                                         tol_primal, max_outer, max_inner, inner_tol_floor,
                                         inner_tol_factor, fixed_tol, int(warm_start),
                                         None if yb is None else _ptr(yb))
        if not self.h:
            lib.check(-1)
        self.N = lib.lib.ref_admm_size(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.lib.ref_admm_destroy(self.h)
            self.h = None

    def krylov_init(self, rhs):
        """pcg start (x = 0): returns the iteration state dict."""
        st = {k: np.zeros(self.N) for k in ("x", "r", "z", "p", "q")}
        st["rz"] = np.zeros(1)
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        self.L.check(self.L.lib.ref_admm_krylov_init(self.h, _ptr(rhs), _ptr(st["r"]), _ptr(st["z"]),
                                                     _ptr(st["p"]), _ptr(st["rz"])))
        return st

    def krylov_iteration(self, st):
        """One iteration of the reference pcg loop body; returns (pq, |r|, rz)."""
        out = np.zeros(3)
        self.L.check(self.L.lib.ref_admm_krylov_iteration(
            self.h, _ptr(st["x"]), _ptr(st["r"]), _ptr(st["z"]), _ptr(st["p"]), _ptr(st["q"]),
            _ptr(st["rz"]), _ptr(out)))
        return out


# --------------------------------------------------------------------------
# The generalized C restatement (oracle/build/liboracle.so)
# --------------------------------------------------------------------------
class PortLib(_Lib):
    so_path = PORT_SO
    err_fn = "or_last_error"

    def __init__(self):
        super().__init__()
        L = self.lib
        for name in ("or_op_create", "or_pc_assemble", "or_admm_create"):
            getattr(L, name).restype = C.c_void_p
        L.or_op_create.argtypes = [C.c_int] * 3 + [_dp] * 6 + [C.c_double]
        L.or_op_destroy.argtypes = [C.c_void_p]
        L.or_op_apply.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        L.or_op_apply_direct.argtypes = [C.c_void_p, _dp, _dp, C.c_int]
        L.or_pc_assemble.argtypes = [C.c_void_p] + [C.c_double] * 3
        L.or_pc_destroy.argtypes = [C.c_void_p]
        L.or_pc_solve.argtypes = [C.c_void_p, _dp, _dp]
        L.or_pc_lam_s.argtypes = [C.c_void_p, _dp]
        L.or_pc_eigs.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.or_admm_create.argtypes = ([C.c_void_p, C.c_void_p] + [C.c_double] * 8
                                     + [C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, _dp])
        L.or_admm_destroy.argtypes = [C.c_void_p]
        L.or_admm_size.argtypes = [C.c_void_p]
        L.or_admm_size.restype = C.c_size_t
        for name in ("or_admm_get", "or_admm_set"):
            getattr(L, name).argtypes = [C.c_void_p, C.c_int, _dp]
        L.or_admm_apply_S.argtypes = [C.c_void_p, _dp, _dp]
        L.or_admm_build_rhs.argtypes = [C.c_void_p, _dp, _dp]
        L.or_admm_pcg.argtypes = [C.c_void_p, _dp, _dp, C.c_double, C.c_int, _dp]
        L.or_admm_step.argtypes = [C.c_void_p, _dp]
        L.or_admm_dual_inf.argtypes = [C.c_void_p, _dp]
        L.or_admm_objective.argtypes = [C.c_void_p, _dp]
        L.or_frac_coeffs.argtypes = [C.c_double, C.c_int, _dp]
        L.or_build_riesz.argtypes = [C.c_double, C.c_int, C.c_double, _dp]
        L.or_build_caputo.argtypes = [C.c_double, C.c_int, C.c_double, _dp, _dp]
        L.or_embed_symbol.argtypes = [C.c_int, _dp, _dp, C.c_int, _dp]
        L.or_tchan.argtypes = [C.c_int, _dp, _dp, _dp, _dp]
        L.or_set_threads.argtypes = [C.c_int]
        L.or_get_threads.restype = C.c_int

    def frac_coeffs(self, order, count):
        out = np.zeros(count)
        self.check(self.lib.or_frac_coeffs(order, count, _ptr(out)))
        return out

    def set_threads(self, t):
        """Fibre-parallel operator / preconditioner loops (bit-identical for
        any count; reductions stay serial)."""
        self.lib.or_set_threads(int(t))

    def get_threads(self):
        return int(self.lib.or_get_threads())

    def build_riesz(self, beta, n, h):
        col = np.zeros(n)
        self.check(self.lib.or_build_riesz(beta, n, h, _ptr(col)))
        return col, col.copy()

    def build_caputo(self, alpha, n, h):
        col, row = np.zeros(n), np.zeros(n)
        self.check(self.lib.or_build_caputo(alpha, n, h, _ptr(col), _ptr(row)))
        return col, row

    def tchan(self, col, row):
        n = len(col)
        col, row = (np.ascontiguousarray(v, dtype=np.float64) for v in (col, row))
        fc, eig = np.zeros(n), np.zeros(2 * n)
        self.check(self.lib.or_tchan(n, _ptr(col), _ptr(row), _ptr(fc), _ptr(eig)))
        return fc, eig[0::2] + 1j * eig[1::2]

    def op(self, shape, time, r1, r2, psi):
        nt, n1, n2 = shape
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (*time, *r1, *r2)]
        h = self.lib.or_op_create(nt, n1, n2, *[_ptr(a) for a in arrs], psi)
        if not h:
            self.check(-1)
        return PortOp(self, h, shape, psi)


class PortOp:
    def __init__(self, lib, h, shape, psi):
        self.L, self.h, self.shape, self.psi = lib, h, tuple(shape), psi
        self.size = shape[0] * shape[1] * shape[2]

    def __del__(self):
        if getattr(self, "h", None):
            self.L.lib.or_op_destroy(self.h)
            self.h = None

    def apply(self, x, adjoint=False, direct=False):
        x = np.ascontiguousarray(x, dtype=np.float64)
        assert x.size == self.size
        out = np.zeros(self.size)
        fn = self.L.lib.or_op_apply_direct if direct else self.L.lib.or_op_apply
        self.L.check(fn(self.h, _ptr(x), _ptr(out), int(adjoint)))
        return out

    def assemble_precond(self, rho, delta, gamma):
        h = self.L.lib.or_pc_assemble(self.h, rho, delta, gamma)
        if not h:
            self.L.check(-1)
        return PortPc(self.L, h, self, rho, delta, gamma)


class PortPc:
    def __init__(self, lib, h, op, rho, delta, gamma):
        self.L, self.h, self.op = lib, h, op
        self.rho, self.delta, self.gamma = rho, delta, gamma
        self.size = op.size

    def __del__(self):
        if getattr(self, "h", None):
            self.L.lib.or_pc_destroy(self.h)
            self.h = None

    def solve(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(self.size)
        self.L.check(self.L.lib.or_pc_solve(self.h, _ptr(r), _ptr(z)))
        return z

    def lam_s(self):
        out = np.zeros(self.size)
        self.L.check(self.L.lib.or_pc_lam_s(self.h, _ptr(out)))
        return out

    def eigs(self):
        nt, n1, n2 = self.op.shape
        a, b, c = np.zeros(2 * nt), np.zeros(2 * n1), np.zeros(2 * n2)
        self.L.check(self.L.lib.or_pc_eigs(self.h, _ptr(a), _ptr(b), _ptr(c)))
        return tuple(v[0::2] + 1j * v[1::2] for v in (a, b, c))


class PortAdmm(_AdmmBase):
    pfx = "or_"

    def __init__(self, lib: PortLib, op: PortOp, pc: PortPc, gamma, rho, delta, y_lo=-math.inf,
                 y_hi=math.inf, u_lo=-math.inf, u_hi=math.inf, tol_primal=1e-4, max_inner=400,
                 inner_tol_floor=1e-4, inner_tol_factor=0.05, fixed_tol=0.0, warm_start=False,
                 ybar=None):
        self.L, self._keep = lib, (op, pc)
        yb = None if ybar is None else np.ascontiguousarray(ybar, dtype=np.float64)
        self.h = lib.lib.or_admm_create(op.h, pc.h, gamma, rho, delta, y_lo, y_hi, u_lo, u_hi,
                                        tol_primal, max_inner, inner_tol_floor, inner_tol_factor,
                                        fixed_tol, int(warm_start),
                                        None if yb is None else _ptr(yb))
        self.N = lib.lib.or_admm_size(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.lib.or_admm_destroy(self.h)
            self.h = None

    def pcg(self, rhs, x=None, tol=1e-8, max_inner=400):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.zeros(self.N) if x is None else np.ascontiguousarray(x, dtype=np.float64).copy()
        res = np.zeros(3)
        self.L.check(self.L.lib.or_admm_pcg(self.h, _ptr(rhs), _ptr(x), tol, max_inner, _ptr(res)))
        return x, dict(iterations=int(res[0]), converged=bool(res[1]), rel_residual=res[2])

    def step(self):
        rec = np.zeros(8)
        self.L.check(self.L.lib.or_admm_step(self.h, _ptr(rec)))
        return dict(iter=int(rec[0]), r_eq=rec[1], r_y=rec[2], r_u=rec[3], dual_inf=rec[4],
                    inner_iters=int(rec[5]), inner_tol=rec[6], converged=bool(rec[7]))


_REF = None
_PORT = None


def ref_lib() -> RefLib:
    global _REF
    if _REF is None:
        _REF = RefLib()
    return _REF


def port_lib() -> PortLib:
    global _PORT
    if _PORT is None:
        _PORT = PortLib()
    return _PORT


# --------------------------------------------------------------------------
# BASELINE config -> reference mapping, via the
# reference's own coefficient builders.
# --------------------------------------------------------------------------
@dataclass
class Shape:
    nt: int
    n1: int
    n2: int

    @property
    def N(self):
        return self.nt * self.n1 * self.n2

    def tuple(self):
        return (self.nt, self.n1, self.n2)


def implicit_euler(nt, h_t):
    """GL alpha=1 time factor: col=(1,-1,0..)/h_t, row=(1,0,..)/h_t (App. A.1)."""
    col = np.zeros(nt)
    row = np.zeros(nt)
    col[0] = 1.0 / h_t
    if nt > 1:
        col[1] = -1.0 / h_t
    row[0] = col[0]
    return col, row


def riesz(beta, n, h, d=1.0):
    col, row = ref_lib().build_riesz(beta, n, h)
    return col * d, row * d


def randn(seed, count):
    return ref_lib().randn(seed, count)


def synthetic_ybar(kind, shape: Shape, seed=1, sigma=0.01):
    """BASELINE target states at x=(i+1)h_x, t=(k+1)h_t plus sigma*N(0,1)."""
    nt, n1, n2 = shape.tuple()
    ht = 1.0 / nt
    x1 = (np.arange(n1) + 1.0) / (n1 + 1)
    x2 = (np.arange(n2) + 1.0) / (n2 + 1)
    t = (np.arange(nt) + 1.0) * ht
    T, X1, X2 = np.meshgrid(t, x1, x2, indexing="ij")
    if kind == "sin":
        base = np.sin(np.pi * X1) * np.sin(np.pi * X2) * np.exp(T)
    elif kind == "bump":
        base = np.exp(-50.0 * ((X2 - 0.5) ** 2 + (X1 - 0.5) ** 2)) * (1.0 + T)
    else:
        raise ValueError(kind)
    return (base.ravel() + sigma * randn(seed, shape.N)).astype(np.float64)


def baseline_problem(name: str, shape: Shape | None = None):
    """BASELINE.json configs C0, C2, C3, C4 (full solves) as reference inputs."""
    cfgs = {
        "C0": dict(shape=Shape(32, 32, 32), ax=1.5, ay=1.5, dx=1.0, dy=1.0, gamma=1e-4,
                   u=(-2.0, 1.5), y=(-math.inf, math.inf), ybar="sin"),
        "C2": dict(shape=Shape(256, 256, 256), ax=1.5, ay=1.5, dx=1.0, dy=1.0, gamma=1e-5,
                   u=(-1.0, 1.0), y=(-math.inf, math.inf), ybar="sin"),
        "C3": dict(shape=Shape(128, 512, 512), ax=1.2, ay=1.8, dx=1.0, dy=0.5, gamma=1e-6,
                   u=(-5.0, 5.0), y=(0.0, 0.8), ybar="bump"),
        "C4": dict(shape=Shape(128, 1024, 1024), ax=1.5, ay=1.5, dx=1.0, dy=1.0, gamma=1e-4,
                   u=(-1.0, 1.0), y=(-math.inf, math.inf), ybar="sin"),
    }
    c = dict(cfgs[name])
    if shape is not None:
        c["shape"] = shape
    s = c["shape"]
    ht = 1.0 / s.nt
    h1 = 1.0 / (s.n1 + 1)
    h2 = 1.0 / (s.n2 + 1)
    time = implicit_euler(s.nt, ht)
    r2 = riesz(c["ax"], s.n2, h2, c["dx"])   # BASELINE x -> reference x2 (innermost)
    r1 = riesz(c["ay"], s.n1, h1, c["dy"])   # BASELINE y -> reference x1
    psi = min(ht ** 1.0, h2 ** c["ax"], h1 ** c["ay"])
    c.update(time=time, r1=r1, r2=r2, psi=psi, rho=1.0, delta=1.0, krylov_tol=1e-8,
             tol_primal=1e-6, max_inner=400)
    return c


def spatial_precond_solve(shape, lam_x1, lam_x2, r):
    """BASELINE C1 preconditioner restated with numpy (pocketfft): per time
    slice z = F^-1 (F r / (lam_x1[i] + lam_x2[j])), the 2-level T. Chan
    circulant of A = I (x) T_x + T_y (x) I.  Independent of
    the GPU's Bluestein Hartley passes."""
    nt, n1, n2 = shape
    R = np.asarray(r, dtype=np.float64).reshape(nt, n1, n2)
    D = np.asarray(lam_x1)[:, None] + np.asarray(lam_x2)[None, :]
    Z = np.fft.ifft2(np.fft.fft2(R, axes=(1, 2)) / D, axes=(1, 2))
    return np.ascontiguousarray(Z.real).ravel()


def circulant_dense(first_col):
    """Dense circulant with the given first column (C[i, j] = c[(i - j) mod n])."""
    c = np.asarray(first_col)
    n = c.size
    idx = (np.arange(n)[:, None] - np.arange(n)[None, :]) % n
    return c[idx]

