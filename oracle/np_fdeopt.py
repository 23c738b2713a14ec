"""oracle/np_fdeopt.py — TEST INFRASTRUCTURE (CPU checker; never the product).

A numpy restatement of the reference hot path with an INDEPENDENT FFT
backend (numpy's pocketfft instead of the FFTW3 shim that oracle/_ref and
oracle/build share).  Its only job is to measure the cross-implementation
noise floor of a full ADMM solve (SURVEY.md §7 "hard parts"): two correct
fp64 implementations whose FFTs round differently drift apart over 11k ADMM
steps, and the difference between this solve and the reference's is the
floor below which no GPU-vs-reference residual gate can be met.

Restates (file:line under /root/reference/proj/src):
  toeplitz.cpp:46-58   embed_symbol (first column of the 2n circulant)
  toeplitz.cpp:124-182 apply_mode / apply (mode-wise embedding by FFT)
  circulant.cpp:10-20  tchan; 22-26 circulant_eigs; 76-90 assemble_precond
  circulant.cpp:49-67  CirculantPreconditioner::solve
  admm.cpp:87-98 apply_S, 100-119 build_rhs, 121-169 pcg, 171-233 updates,
  residuals and dual_infeasibility, 245-277 AdmmDriver::step.
"""
from __future__ import annotations

import math

import numpy as np


def _embed(col, row, transpose=False):
    """toeplitz.cpp:46-58: c = (t_0..t_{n-1}, 0, t_{-(n-1)}..t_{-1}); transpose swaps."""
    if transpose:
        col, row = row, col
    n = len(col)
    c = np.zeros(2 * n)
    c[:n] = col
    c[n + 1:] = row[1:][::-1]
    return np.fft.rfft(c)


def _tchan_eigs(col, row):
    """circulant.cpp:10-26: c_i = ((n-i) t_i + i t_{-(n-i)}) / n, eigenvalues by DFT."""
    n = len(col)
    c = np.empty(n)
    c[0] = col[0]
    for i in range(1, n):
        c[i] = ((n - i) * col[i] + i * row[n - i]) / n
    return np.fft.fft(c)


class NpOperator:
    """ConstraintOperator (toeplitz.cpp:87-189) for (n_t, n_x1, n_x2) shapes."""

    def __init__(self, shape, time, r1, r2, psi):
        self.shape = tuple(shape)
        self.time, self.r1, self.r2 = time, r1, r2
        self.psi = psi
        self.sym = {("t", False): _embed(*time), ("t", True): _embed(*time, transpose=True),
                    1: _embed(*r1), 2: _embed(*r2)}

    @property
    def size(self):
        return self.shape[0] * self.shape[1] * self.shape[2]

    @staticmethod
    def _mode(x, axis, sym):
        n = x.shape[axis]
        spec = np.fft.rfft(x, n=2 * n, axis=axis)
        shp = [1, 1, 1]
        shp[axis] = n + 1
        y = np.fft.irfft(spec * sym.reshape(shp), n=2 * n, axis=axis)
        return np.take(y, np.arange(n), axis=axis)

    def apply(self, x, adjoint=False):
        X = np.asarray(x, dtype=np.float64).reshape(self.shape)
        out = self.psi * self._mode(X, 0, self.sym[("t", adjoint)])
        out -= self.psi * self._mode(X, 1, self.sym[1])
        out -= self.psi * self._mode(X, 2, self.sym[2])
        return out.ravel()


class NpPrecond:
    """CirculantPreconditioner (circulant.cpp:28-90) with the T. Chan eigenvalues."""

    def __init__(self, op: NpOperator, rho, delta, gamma):
        psi = op.psi
        lt = _tchan_eigs(*op.time)
        l1 = _tchan_eigs(*op.r1)
        l2 = _tchan_eigs(*op.r2)
        lam_b = psi * (lt[:, None, None] - (l1[None, :, None] + l2[None, None, :]))
        m2 = 1.0 / (rho * (gamma / (psi * psi) + 1.0 / delta)) + delta / rho
        self.lam_s = rho * (1.0 + 1.0 / delta) + np.abs(lam_b) ** 2 / m2
        self.shape = op.shape

    def solve(self, r):
        R = np.asarray(r, dtype=np.float64).reshape(self.shape)
        return np.fft.ifftn(np.fft.fftn(R) / self.lam_s).real.ravel()


class NpAdmm:
    """AdmmDriver::step (admm.cpp:245-277) with the BASELINE mapping (fixed
    Krylov tol, injected ybar), the same sequence as oracle/fdeopt_oracle.c."""

    def __init__(self, op, pc, gamma, rho, delta, y_lo=-math.inf, y_hi=math.inf, u_lo=-math.inf,
                 u_hi=math.inf, tol_primal=1e-6, max_inner=400, fixed_tol=1e-8, ybar=None):
        self.op, self.pc = op, pc
        N = op.size
        nt = op.shape[0]
        psi = op.psi
        self.rho, self.delta, self.psi = rho, delta, psi
        self.tol_primal, self.max_inner, self.fixed_tol = tol_primal, max_inner, fixed_tol
        self.y_lo, self.y_hi, self.v_lo, self.v_hi = y_lo, y_hi, psi * u_lo, psi * u_hi
        j = np.ones(N)
        j[(nt - 1) * (N // nt):] = 0.5
        self.diag_j = j
        self.diag_j2 = gamma / (psi * psi) * j
        self.a2_inv = 1.0 / (rho * (self.diag_j2 + 1.0 / delta))
        self.m2 = self.a2_inv + delta / rho
        self.ybar = np.zeros(N) if ybar is None else np.asarray(ybar, dtype=np.float64).copy()
        for f in ("y", "v", "z_y", "z_v", "p", "w_y", "w_v", "By"):
            setattr(self, f, np.zeros(N))
        self.iteration = 0

    def apply_S(self, x):
        bx = self.op.apply(x) / self.m2
        return self.rho * (self.diag_j + 1.0 / self.delta) * x + self.op.apply(bx, True)

    def build_rhs(self):
        rho, delta = self.rho, self.delta
        r = (delta / rho) * self.p + self.a2_inv * (rho * (-self.w_v + self.z_v / delta)
                                                    + (1.0 - rho) * self.p)
        tmp = (1.0 - rho) * self.p - r / self.m2
        rhs = self.op.apply(tmp, True) + rho * (self.diag_j * self.ybar - self.w_y + self.z_y / delta)
        return rhs, r

    def pcg(self, rhs, tol, max_inner):
        nb = math.sqrt(rhs @ rhs)
        x = np.zeros_like(rhs)
        if nb == 0.0:
            return x, 0, True
        r = rhs.copy()
        z = self.pc.solve(r)
        p = z.copy()
        rz = r @ z
        for it in range(1, max_inner + 1):
            q = self.apply_S(p)
            pq = p @ q
            if not math.isfinite(pq) or pq <= 0.0:
                raise RuntimeError("pcg: operator lost positive definiteness")
            al = rz / pq
            x += al * p
            r -= al * q
            rn = math.sqrt(r @ r)
            if rn <= tol * nb:
                r = rhs - self.apply_S(x)
                rn = math.sqrt(r @ r)
                if rn <= tol * nb:
                    return x, it, True
            z = self.pc.solve(r)
            rz_next = r @ z
            beta = rz_next / rz
            rz = rz_next
            p = z + beta * p
        return x, max_inner, False

    def step(self):
        rho, delta = self.rho, self.delta
        rhs, r_cache = self.build_rhs()
        self.y, its, _ = self.pcg(rhs, self.fixed_tol, self.max_inner)
        self.By = self.op.apply(self.y)
        pt = (self.By + r_cache) / self.m2
        self.v = self.a2_inv * (-pt - rho * self.w_v + (rho / delta) * self.z_v + (1.0 - rho) * self.p)
        self.z_y = np.clip(self.y + delta * self.w_y, self.y_lo, self.y_hi)
        self.z_v = np.clip(self.v + delta * self.w_v, self.v_lo, self.v_hi)
        step = rho / delta
        self.p = self.p + step * (self.By + self.v)
        self.w_y = self.w_y + step * (self.y - self.z_y)
        self.w_v = self.w_v + step * (self.v - self.z_v)
        self.iteration += 1
        r_eq = float(np.abs(self.By + self.v).max())
        r_y = float(np.abs(self.y - self.z_y).max())
        r_u = float(np.abs(self.v - self.z_v).max()) / self.psi
        btp = self.op.apply(self.p, True)
        dinf = max(float(np.abs(self.diag_j * (self.y - self.ybar) + btp + self.w_y).max()),
                   float(np.abs(self.diag_j2 * self.v + self.p + self.w_v).max()))
        conv = r_eq <= self.tol_primal and r_y <= self.tol_primal and r_u <= self.tol_primal
        return dict(iter=self.iteration, r_eq=r_eq, r_y=r_y, r_u=r_u, dual_inf=dinf,
                    inner_iters=its, converged=conv)

    def objective(self):
        d = self.y - self.ybar
        return 0.5 * float(self.diag_j @ (d * d)) + 0.5 * float(self.diag_j2 @ (self.v * self.v))
