"""BASELINE.json workloads mapped onto the reference's problem.

  axes: BASELINE x -> reference x2 (innermost), BASELINE y -> reference x1
  time: implicit Euler = GL alpha=1 bidiagonal, h_t = 1/n_t, t_k = (k+1) h_t
  space: h = 1/(n+1), x_i = (i+1) h;  psi = min(h_t, h_x2^ax, h_x1^ay) (d excluded)
  ADMM: penalty 1 -> delta = rho = 1; Krylov tol fixed 1e-8; tol_primal 1e-6
  preconditioner: the reference's T. Chan circulant (only one it ships)
  desired state: seeded noise from std::mt19937_64(seed) + normal_distribution
"""
from __future__ import annotations

import math

import numpy as np

CONFIGS = {
    # name: (nt, n1, n2), ax (x2), ay (x1), dx, dy, gamma, u-box, y-box, ybar kind
    "C0": dict(shape=(32, 32, 32), ax=1.5, ay=1.5, dx=1.0, dy=1.0, gamma=1e-4, u=(-2.0, 1.5),
               y=(-math.inf, math.inf), ybar="sin"),
    "C2": dict(shape=(256, 256, 256), ax=1.5, ay=1.5, dx=1.0, dy=1.0, gamma=1e-5, u=(-1.0, 1.0),
               y=(-math.inf, math.inf), ybar="sin"),
    "C3": dict(shape=(128, 512, 512), ax=1.2, ay=1.8, dx=1.0, dy=0.5, gamma=1e-6, u=(-5.0, 5.0),
               y=(0.0, 0.8), ybar="bump"),
    "C4": dict(shape=(128, 1024, 1024), ax=1.5, ay=1.5, dx=1.0, dy=1.0, gamma=1e-4,
               u=(-1.0, 1.0), y=(-math.inf, math.inf), ybar="sin"),
}


def baseline_config(name: str, shape=None) -> dict:
    from .api import build_riesz, implicit_euler
    c = dict(CONFIGS[name])
    if shape is not None:
        c["shape"] = tuple(shape)
    nt, n1, n2 = c["shape"]
    ht, h1, h2 = 1.0 / nt, 1.0 / (n1 + 1), 1.0 / (n2 + 1)
    time = implicit_euler(nt, ht)
    c2, r2 = build_riesz(c["ax"], n2, h2)
    c1, r1 = build_riesz(c["ay"], n1, h1)
    c.update(time=time, x2=(c2 * c["dx"], r2 * c["dx"]), x1=(c1 * c["dy"], r1 * c["dy"]),
             psi=min(ht ** 1.0, h2 ** c["ax"], h1 ** c["ay"]), rho=1.0, delta=1.0,
             krylov_tol=1e-8, tol_primal=1e-6, max_inner=400, name=name)
    return c


def synthetic_ybar(kind: str, shape, seed: int = 1, sigma: float = 0.01) -> np.ndarray:
    from .api import randn
    nt, n1, n2 = shape
    t = (np.arange(nt) + 1.0) / nt
    x1 = (np.arange(n1) + 1.0) / (n1 + 1)
    x2 = (np.arange(n2) + 1.0) / (n2 + 1)
    T, X1, X2 = np.meshgrid(t, x1, x2, indexing="ij")
    if kind == "sin":
        base = np.sin(np.pi * X1) * np.sin(np.pi * X2) * np.exp(T)
    elif kind == "bump":
        base = np.exp(-50.0 * ((X2 - 0.5) ** 2 + (X1 - 0.5) ** 2)) * (1.0 + T)
    else:
        raise ValueError(kind)
    return base.ravel() + sigma * randn(seed, nt * n1 * n2)


def make_problem(name: str, shape=None, ctx=None, seed: int = 1, ybar=None):
    """Operator, preconditioner and ADMM driver of a BASELINE config."""
    from .api import AdmmConfig, AdmmDriver, ConstraintOperator, assemble_precond
    c = baseline_config(name, shape)
    op = ConstraintOperator(c["time"], c["x1"], c["x2"], c["psi"], ctx=ctx)
    pc = assemble_precond(op, c["rho"], c["delta"], c["gamma"])
    cfg = AdmmConfig(delta=c["delta"], rho=c["rho"], tol_primal=c["tol_primal"], max_outer=100000,
                     max_inner=c["max_inner"], fixed_krylov_tol=c["krylov_tol"])
    yb = synthetic_ybar(c["ybar"], c["shape"], seed) if ybar is None else ybar
    drv = AdmmDriver(op, pc, c["gamma"], cfg, y_lo=c["y"][0], y_hi=c["y"][1], u_lo=c["u"][0],
                     u_hi=c["u"][1], ybar=yb)
    return c, op, pc, drv


# BASELINE C1 operator microbenchmark: A = I (x) T_x + T_y (x) I on every
# slice, T_x = Riesz(1.3) on x2, T_y = Riesz(1.7) on x1, h = 1/(n + 1); no psi,
# no time term.  Mapped onto the ConstraintOperator with
# psi = -1 and a zero time factor: out = -psi (L1 + L2) x = (T_y + T_x) x.
C1 = dict(shape=(256, 1023, 1023), ax=1.3, ay=1.7)


def c1_factors(shape=None):
    from .api import build_riesz
    nt, n1, n2 = tuple(shape) if shape is not None else C1["shape"]
    tx = build_riesz(C1["ax"], n2, 1.0 / (n2 + 1))
    ty = build_riesz(C1["ay"], n1, 1.0 / (n1 + 1))
    time = (np.zeros(nt), np.zeros(nt))
    return (nt, n1, n2), time, ty, tx


def make_c1(shape=None, ctx=None):
    """C1 operator and its 2-level spatial T. Chan preconditioner."""
    from .api import ConstraintOperator, assemble_spatial_precond
    shp, time, ty, tx = c1_factors(shape)
    op = ConstraintOperator(time, ty, tx, -1.0, ctx=ctx)
    return op, assemble_spatial_precond(op)

