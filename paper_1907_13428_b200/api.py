"""Host-side mirror of the reference interface over the C ABI (include/fdg.h).

Names, argument meaning and error behaviour follow the reference:
  ConstraintOperator.apply      toeplitz.hpp:55-57   (ValueError == std::invalid_argument)
  assemble_precond / .solve     circulant.hpp:43, 63-64
  AdmmDriver.step / state       admm.hpp:128-150
  AdmmDriver.pcg / apply_S      admm.hpp:79-80, 97-98
  solve                         admm.hpp:154-155, admm.cpp:279-324
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import FdgError, check, lib

_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _addr(x) -> int:
    """Device address of a torch tensor or an int."""
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


# ------------------------------------------------------------- 1-D setup
def frac_coeffs(order: float, count: int) -> np.ndarray:
    out = np.zeros(count)
    check(lib.fdg_frac_coeffs(order, count, _ptr(out)))
    return out


def build_riesz(beta: float, n: int, h: float):
    col, row = np.zeros(n), np.zeros(n)
    check(lib.fdg_build_riesz(beta, n, h, _ptr(col), _ptr(row)))
    return col, row


def build_caputo(alpha: float, n: int, h: float):
    col, row = np.zeros(n), np.zeros(n)
    check(lib.fdg_build_caputo(alpha, n, h, _ptr(col), _ptr(row)))
    return col, row


def implicit_euler(nt: int, h_t: float):
    """Implicit Euler time factor = Grunwald-Letnikov alpha = 1 bidiagonal
    (SURVEY.md Appendix A.1): col = (1, -1, 0, ..)/h_t, row = (1, 0, ..)/h_t."""
    col, row = np.zeros(nt), np.zeros(nt)
    col[0] = 1.0 / h_t
    if nt > 1:
        col[1] = -1.0 / h_t
    row[0] = col[0]
    return col, row


def tchan(col, row):
    col, row = _f64(col), _f64(row)
    n = col.size
    fc, eig = np.zeros(n), np.zeros(2 * n)
    check(lib.fdg_tchan(n, _ptr(col), _ptr(row), _ptr(fc), _ptr(eig)))
    return fc, eig[0::2] + 1j * eig[1::2]


def randn(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count)
    check(lib.fdg_randn(seed, count, _ptr(out)))
    return out


# --------------------------------------------------------------- context
class Context:
    def __init__(self, device: int = 0, stream: int | None = None):
        h = C.c_void_p()
        check(lib.fdg_ctx_create(device, stream, C.byref(h)))
        self.h = h.value
        self.device = device

    def __del__(self):
        if getattr(self, "h", None):
            lib.fdg_ctx_destroy(self.h)
            self.h = None

    @property
    def stream(self) -> int:
        return lib.fdg_ctx_stream(self.h)

    @property
    def launch_count(self) -> int:
        return int(lib.fdg_ctx_launch_count(self.h))

    def synchronize(self):
        check(lib.fdg_ctx_synchronize(self.h))


_default_ctx: Context | None = None


def set_pcg_graph_nmax(nmax: int) -> int:
    """Size threshold of the graph-driven PCG iterations (fdg_set_pcg_graph_nmax);
    returns the previous value.  0 disables them."""
    prev = C.c_longlong()
    check(lib.fdg_set_pcg_graph_nmax(int(nmax), C.byref(prev)))
    return int(prev.value)


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


# -------------------------------------------------------------- operator
class ConstraintOperator:
    """B = psi (T_t x I x I - I x T_1 x I - I x I x T_2) on an (n_t, n_x1, n_x2) grid.

    ``time``, ``x1``, ``x2`` are ToeplitzSpec1D pairs (col, row)
    (toeplitz.hpp:14-19, explicit-factor ctor toeplitz.cpp:87-101)."""

    def __init__(self, time, x1, x2, psi: float, shape=None, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        tcol, trow = (_f64(v) for v in time)
        c1, r1 = (_f64(v) for v in x1)
        c2, r2 = (_f64(v) for v in x2)
        nt, n1, n2 = tcol.size, c1.size, c2.size
        if shape is not None and tuple(shape) != (nt, n1, n2):
            raise ValueError("ConstraintOperator: factor size mismatch")
        if trow.size != nt or r1.size != n1 or r2.size != n2:
            raise ValueError("ConstraintOperator: factor size mismatch")
        h = C.c_void_p()
        check(lib.fdg_op_create(self.ctx.h, nt, n1, n2, _ptr(tcol), _ptr(trow), _ptr(c1), _ptr(r1),
                                _ptr(c2), _ptr(r2), psi, C.byref(h)))
        self.h = h.value
        self.shape = (nt, n1, n2)
        self.time, self.x1, self.x2 = (tcol, trow), (c1, r1), (c2, r2)

    def __del__(self):
        if getattr(self, "h", None):
            lib.fdg_op_destroy(self.h)
            self.h = None

    @property
    def size(self) -> int:
        return int(lib.fdg_op_size(self.h))

    @property
    def psi(self) -> float:
        return float(lib.fdg_op_psi(self.h))

    def apply(self, x, adjoint: bool = False, out_size: int | None = None) -> np.ndarray:
        x = _f64(x)
        out = np.zeros(self.size if out_size is None else out_size)
        check(lib.fdg_op_apply_host(self.h, _ptr(x), x.size, _ptr(out), out.size, int(adjoint)))
        return out

    def apply_dev(self, x, out, adjoint: bool = False) -> None:
        check(lib.fdg_op_apply(self.h, _addr(x), _addr(out), int(adjoint)))


class CirculantPreconditioner:
    """S~ = rho(1 + 1/delta) I + C3(B)^T C3(B)/m2 (circulant.hpp:28-61)."""

    def __init__(self, h, shape, ctx, keep=None):
        self.h, self.shape, self.ctx, self._keep = h, tuple(shape), ctx, keep

    @classmethod
    def from_eigs(cls, lam_t, lam_x1, lam_x2, psi, rho, delta, gamma, ctx: Context | None = None):
        ctx = ctx or default_context()
        arrs = [_f64(np.stack([np.real(v), np.imag(v)], -1).ravel()) for v in (lam_t, lam_x1, lam_x2)]
        h = C.c_void_p()
        shape = (len(lam_t), len(lam_x1), len(lam_x2))
        check(lib.fdg_pc_create(ctx.h, *shape, *[_ptr(a) for a in arrs], psi, rho, delta, gamma,
                                C.byref(h)))
        return cls(h.value, shape, ctx)

    def __del__(self):
        if getattr(self, "h", None):
            lib.fdg_pc_destroy(self.h)
            self.h = None

    @property
    def size(self) -> int:
        return self.shape[0] * self.shape[1] * self.shape[2]

    def solve(self, r, out_size: int | None = None) -> np.ndarray:
        r = _f64(r)
        z = np.zeros(self.size if out_size is None else out_size)
        check(lib.fdg_pc_solve_host(self.h, _ptr(r), r.size, _ptr(z), z.size))
        return z

    def solve_dev(self, r, z) -> None:
        check(lib.fdg_pc_solve(self.h, _addr(r), _addr(z)))

    def lam_s(self) -> np.ndarray:
        out = np.zeros(self.size)
        check(lib.fdg_pc_lam_s_host(self.h, _ptr(out)))
        return out


def assemble_precond(op: ConstraintOperator, rho: float, delta: float, gamma: float):
    """circulant.cpp:76-90"""
    h = C.c_void_p()
    check(lib.fdg_pc_assemble(op.h, rho, delta, gamma, C.byref(h)))
    return CirculantPreconditioner(h.value, op.shape, op.ctx, keep=op)


class SpatialPreconditioner(CirculantPreconditioner):
    """Per-slice 2-level T. Chan preconditioner of A = I (x) T_x + T_y (x) I
    (BASELINE C1): z = F^-1 (F r / (lam_x1[i] + lam_x2[j])) slice by slice,
    any level sizes up to 1024 (Bluestein Hartley passes)."""

    @classmethod
    def from_eigs(cls, n_t, lam_x1, lam_x2, ctx: Context | None = None):
        ctx = ctx or default_context()
        arrs = [_f64(np.stack([np.real(v), np.imag(v)], -1).ravel()) for v in (lam_x1, lam_x2)]
        h = C.c_void_p()
        shape = (int(n_t), len(lam_x1), len(lam_x2))
        check(lib.fdg_pc2_create(ctx.h, *shape, *[_ptr(a) for a in arrs], C.byref(h)))
        return cls(h.value, shape, ctx)

    def lam_s(self):
        raise ValueError("lam_S exists only for the 3-level CirculantPreconditioner")


def assemble_spatial_precond(op: ConstraintOperator) -> SpatialPreconditioner:
    """2-level T. Chan preconditioner from the operator's spatial factors
    (circulant.cpp:10-26 per level)."""
    h = C.c_void_p()
    check(lib.fdg_pc2_assemble(op.h, C.byref(h)))
    return SpatialPreconditioner(h.value, op.shape, op.ctx, keep=op)


# ------------------------------------------------------------------ ADMM
@dataclass
class AdmmConfig:
    """admm.hpp:14-26, plus the BASELINE fixed Krylov tolerance."""
    delta: float = 0.4
    rho: float = 1.618
    tol_primal: float = 1e-4
    max_outer: int = 500
    inner_tol_floor: float = 1e-4
    inner_tol_factor: float = 0.05
    max_inner: int = 400
    warm_start: bool = False
    fixed_krylov_tol: float = 0.0  # > 0: fixed (BASELINE: 1e-8)


@dataclass
class IterRecord:
    iter: int
    r_eq: float
    r_y: float
    r_u: float
    dual_inf: float
    inner_iters: int
    inner_tol: float
    converged: bool = False
    pcg_converged: bool = True
    pcg_rel_residual: float = 0.0
    pcg_ms: float = 0.0
    step_ms: float = 0.0


@dataclass
class PcgResult:
    iterations: int
    converged: bool
    rel_residual: float
    ms: float = 0.0


class AdmmDriver:
    """AdmmDriver(spec, cfg, op, pc) with the desired state injectable
    (AdmmWork::ybar, admm.hpp:66).  Bounds are in the unscaled control u."""

    def __init__(self, op: ConstraintOperator, pc: CirculantPreconditioner, gamma: float,
                 cfg: AdmmConfig | None = None, y_lo=-math.inf, y_hi=math.inf, u_lo=-math.inf,
                 u_hi=math.inf, ybar=None):
        self.op, self.pc = op, pc
        self.cfg = cfg or AdmmConfig()
        c = self.cfg
        desc = N.AdmmDesc(gamma, c.rho, c.delta, y_lo, y_hi, u_lo, u_hi, c.tol_primal, c.max_outer,
                          c.max_inner, c.inner_tol_floor, c.inner_tol_factor, c.fixed_krylov_tol,
                          int(c.warm_start))
        yb = None if ybar is None else _f64(ybar)
        if yb is not None and yb.size != op.size:
            raise ValueError("AdmmDriver: ybar size mismatch")
        h = C.c_void_p()
        check(lib.fdg_admm_create(op.h, pc.h, C.byref(desc), None if yb is None else _ptr(yb),
                                  C.byref(h)))
        self.h = h.value
        self.N = op.size
        self.psi = op.psi
        self.history: list[IterRecord] = []

    def __del__(self):
        if getattr(self, "h", None):
            lib.fdg_admm_destroy(self.h)
            self.h = None

    def step(self) -> IterRecord:
        rec = N.IterRecord()
        check(lib.fdg_admm_step(self.h, C.byref(rec)))
        r = IterRecord(rec.iter, rec.r_eq, rec.r_y, rec.r_u, rec.dual_inf, rec.inner_iters,
                       rec.inner_tol, bool(rec.converged), bool(rec.pcg_converged),
                       rec.pcg_rel_residual, rec.pcg_ms, rec.step_ms)
        self.history.append(r)
        return r

    def converged(self) -> bool:
        return bool(lib.fdg_admm_converged(self.h))

    def consecutive_stagnations(self) -> int:
        return int(lib.fdg_admm_stagnations(self.h))

    def get(self, name: str) -> np.ndarray:
        out = np.zeros(self.N)
        check(lib.fdg_admm_get(self.h, N.FIELDS[name], _ptr(out)))
        return out

    def set(self, name: str, value) -> None:
        v = _f64(value)
        if v.size != self.N:
            raise ValueError("AdmmDriver.set: size mismatch")
        check(lib.fdg_admm_set(self.h, N.FIELDS[name], _ptr(v)))

    def field_ptr(self, name: str) -> int:
        p = C.c_void_p()
        check(lib.fdg_admm_field_ptr(self.h, N.FIELDS[name], C.byref(p)))
        return p.value

    def state(self) -> dict:
        return {k: self.get(k) for k in ("y", "v", "z_y", "z_v", "p", "w_y", "w_v")}

    # --- free functions of admm.hpp on this driver's work ---------------
    def apply_S_dev(self, x, out) -> None:
        check(lib.fdg_admm_apply_S(self.h, _addr(x), _addr(out)))

    def build_rhs_dev(self, rhs, r_cache=None) -> None:
        check(lib.fdg_admm_build_rhs(self.h, _addr(rhs), None if r_cache is None else _addr(r_cache)))

    def pcg_dev(self, rhs, x, tol: float, max_inner: int) -> PcgResult:
        r = N.PcgResult()
        check(lib.fdg_admm_pcg(self.h, _addr(rhs), _addr(x), tol, max_inner, C.byref(r)))
        return PcgResult(r.iterations, bool(r.converged), r.rel_residual, r.ms)

    def pcg(self, rhs, x=None, tol: float = 1e-8, max_inner: int = 400):
        """Host-buffer pcg (H2D rhs/x, device solve, D2H x).  A contiguous
        float64 `x` is updated in place (pass pinned buffers for full copy
        bandwidth); otherwise a copy is made."""
        rhs = _f64(rhs)
        if x is None:
            x = np.zeros(self.N)
        elif not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous
                  and x.flags.writeable):
            x = _f64(x).copy()
        if rhs.size != self.N or x.size != self.N:
            raise ValueError("pcg: dimension mismatch")
        r = N.PcgResult()
        check(lib.fdg_admm_pcg_host(self.h, _ptr(rhs), _ptr(x), tol, max_inner, C.byref(r)))
        return x, PcgResult(r.iterations, bool(r.converged), r.rel_residual, r.ms)

    def dual_infeasibility(self) -> float:
        out = np.zeros(1)
        check(lib.fdg_admm_dual_inf(self.h, _ptr(out)))
        return float(out[0])

    def objective(self) -> float:
        out = np.zeros(1)
        check(lib.fdg_admm_objective(self.h, _ptr(out)))
        return float(out[0])

    def profile_passes(self, reps: int = 10) -> dict:
        ms, by = np.zeros(len(N.PASS_NAMES)), np.zeros(len(N.PASS_NAMES))
        check(lib.fdg_admm_profile_passes(self.h, reps, _ptr(ms), _ptr(by)))
        return {n: dict(ms=float(m), bytes=float(b)) for n, m, b in zip(N.PASS_NAMES, ms, by)}

    def debug_get(self, which: str):
        names = dict(r=0, z=1, p=2, u=3, w=4, vp=5, scalars=-1)
        out = np.zeros(32 if which == "scalars" else self.N)
        check(lib.fdg_admm_debug_get(self.h, names[which], _ptr(out)))
        return out

    # host conveniences used by the parity tests (device work + staging)
    def apply_S(self, x) -> np.ndarray:
        import torch
        xd = torch.from_numpy(_f64(x)).cuda()
        out = torch.empty_like(xd)
        torch.cuda.synchronize()
        self.apply_S_dev(xd, out)
        self.op.ctx.synchronize()
        return out.cpu().numpy()

    def build_rhs(self):
        import torch
        rhs = torch.empty(self.N, dtype=torch.float64, device="cuda")
        rc = torch.empty_like(rhs)
        torch.cuda.synchronize()
        self.build_rhs_dev(rhs, rc)
        self.op.ctx.synchronize()
        return rhs.cpu().numpy(), rc.cpu().numpy()


def solve(driver: AdmmDriver, callback=None) -> dict:
    """fdeopt::solve's outer loop (admm.cpp:289-324) over an AdmmDriver:
    stops on convergence or max_outer; 3 consecutive PCG caps raise."""
    t0 = time.perf_counter()
    cfg = driver.cfg
    total_inner = 0
    status = "itercap"
    for _ in range(cfg.max_outer):
        rec = driver.step()
        total_inner += rec.inner_iters
        if callback:
            callback(rec)
        if driver.consecutive_stagnations() >= 3:
            raise FdgError(N.FDG_ENUMERIC,
                           "admm: PCG hit max_inner in 3 consecutive outer iterations", 4)
        if driver.converged():
            status = "converged"
            break
    it = len(driver.history)
    return dict(status=status, iterations=it, pcg_avg=total_inner / it if it else 0.0,
                dual_inf=driver.dual_infeasibility(), objective=driver.objective(),
                wall_seconds=time.perf_counter() - t0, history=driver.history)
