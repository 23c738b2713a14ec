"""The reference's own experiment as a run configuration (f3).

Host-side restatement of the reference's problem specification and config
file format so that its `solve` / `sweep` / `bench` front end
(`paper_1907_13428_b200.cli`) runs on the B200 path:

  * ProblemSpec / AdmmSettings / RunConfig  -- problem.hpp:15-26,
    admm.hpp:14-26, config.hpp:13-25 (defaults and validation messages:
    problem.cpp:9-20, admm.cpp:34-42);
  * parse_config_file / apply_config_entry / parse_bound -- config.cpp:59-138
    (flat `key = value` lines, `#` comments, the same key set and errors);
  * desired_state_at / l2_misfit -- problem.cpp:47-83;
  * solve_spec -- fdeopt::solve (admm.cpp:279-324): ConstraintOperator(spec,
    grid) (Caputo time factor + Riesz factors, toeplitz.cpp:80-84), the T. Chan
    preconditioner, the AdmmDriver with the reference's desired state and
    dynamic inner tolerance, the outer loop, u = v / psi, misfit, dual_inf.
"""
from __future__ import annotations

import copy
import math
from dataclasses import dataclass, field

import numpy as np

RHO_MAX = 1.6180339887498949  # (sqrt(5)+1)/2, admm.cpp:35


class ConfigError(ValueError):
    """std::invalid_argument of the reference (CLI exit code 1)."""


@dataclass
class ProblemSpec:
    """problem.hpp:15-26"""
    alpha: float = 0.7
    beta1: float = 1.3
    beta2: float = 1.3
    gamma: float = 1e-4
    n: int = 8
    y_lo: float = -math.inf
    y_hi: float = math.inf
    u_lo: float = -math.inf
    u_hi: float = math.inf

    def validate(self) -> None:
        """problem.cpp:9-20"""
        if not (0.0 < self.alpha < 1.0):
            raise ConfigError(f"alpha must lie in (0, 1), got {self.alpha:f}")
        if not (1.0 < self.beta1 < 2.0):
            raise ConfigError(f"beta1 must lie in (1, 2), got {self.beta1:f}")
        if not (1.0 < self.beta2 < 2.0):
            raise ConfigError(f"beta2 must lie in (1, 2), got {self.beta2:f}")
        if not (self.gamma > 0.0):
            raise ConfigError("gamma must be positive")
        if self.n < 1:
            raise ConfigError("n must be >= 1")
        if not (self.y_lo < self.y_hi):
            raise ConfigError("state bounds must satisfy y_lo < y_hi")
        if not (self.u_lo < self.u_hi):
            raise ConfigError("control bounds must satisfy u_lo < u_hi")


@dataclass
class AdmmSettings:
    """admm.hpp:14-26 (the reference's AdmmConfig)."""
    delta: float = 0.4
    rho: float = 1.618
    tol_primal: float = 1e-4
    max_outer: int = 500
    inner_tol_floor: float = 1e-4
    inner_tol_factor: float = 0.05
    max_inner: int = 400
    warm_start: bool = False

    def validate(self) -> None:
        """admm.cpp:34-42"""
        if not (0.0 < self.rho < RHO_MAX):
            raise ConfigError("rho must lie in (0, (sqrt(5)+1)/2)")
        if not (self.delta > 0.0):
            raise ConfigError("delta must be positive")
        if not (self.tol_primal > 0.0) or not (self.inner_tol_floor > 0.0) or not (self.inner_tol_factor > 0.0):
            raise ConfigError("tolerances must be positive")
        if self.max_outer < 1 or self.max_inner < 1:
            raise ConfigError("iteration caps must be >= 1")


@dataclass
class RunConfig:
    """config.hpp:13-25"""
    spec: ProblemSpec = field(default_factory=ProblemSpec)
    admm: AdmmSettings = field(default_factory=AdmmSettings)
    out_dir: str = ""
    format: str = "csv"
    delta_sweep: list = field(default_factory=list)
    n_sweep: list = field(default_factory=list)
    alpha_sweep: list = field(default_factory=list)
    seed: int = 0
    dump_solution: bool = False
    workers: int = 1

    def copy(self) -> "RunConfig":
        return copy.deepcopy(self)


CONFIG_KEYS = ["alpha", "beta1", "beta2", "gamma", "n", "ylo", "yhi", "ulo", "uhi", "delta", "rho", "tol",
               "max_outer", "max_inner", "inner_tol_floor", "inner_tol_factor", "warm_start", "out", "format",
               "delta_sweep", "n_sweep", "alpha_sweep", "seed", "dump", "workers"]  # config.cpp:69-77


def _parse_double(key: str, value: str) -> float:
    """std::stod that must consume the whole string (config.cpp:18-27):
    leading whitespace skipped, decimal / hex / inf / nan spellings."""
    s = value.lstrip()
    try:
        if not s or s != s.rstrip() or "_" in s:
            raise ValueError
        body = s.lstrip("+-").lower()
        return float.fromhex(s) if body.startswith("0x") else float(s)
    except ValueError:
        raise ConfigError(f"config key '{key}' expects a number, got '{value}'") from None


def _parse_int(key: str, value: str) -> int:
    """std::stoi with the whole string consumed (config.cpp:29-39)."""
    v = value.lstrip()
    body = v[1:] if v[:1] in "+-" else v
    if not body.isdigit():
        raise ConfigError(f"config key '{key}' expects an integer, got '{value}'")
    iv = int(v)
    if not (-2 ** 31 <= iv < 2 ** 31):
        raise ConfigError(f"config key '{key}' expects an integer, got '{value}'")
    return iv


def _parse_flag(key: str, value: str) -> bool:
    """config.cpp:41-45"""
    if value in ("true", "1", "yes"):
        return True
    if value in ("false", "0", "no"):
        return False
    raise ConfigError(f"config key '{key}' expects a boolean, got '{value}'")


def _parse_list(key: str, value: str, parse) -> list:
    """config.cpp:47-57"""
    out = [parse(key, item.strip()) for item in value.split(",") if item.strip()]
    if not out:
        raise ConfigError(f"config key '{key}' expects a nonempty list")
    return out


def parse_bound(text: str) -> float:
    """config.cpp:61-66"""
    t = text.strip()
    if t in ("inf", "+inf"):
        return math.inf
    if t == "-inf":
        return -math.inf
    return _parse_double("bound", t)


def apply_config_entry(key: str, value: str, cfg: RunConfig) -> None:
    """config.cpp:80-121"""
    s, a = cfg.spec, cfg.admm
    if key == "alpha":
        s.alpha = _parse_double(key, value)
    elif key == "beta1":
        s.beta1 = _parse_double(key, value)
    elif key == "beta2":
        s.beta2 = _parse_double(key, value)
    elif key == "gamma":
        s.gamma = _parse_double(key, value)
    elif key == "n":
        s.n = _parse_int(key, value)
    elif key == "ylo":
        s.y_lo = parse_bound(value)
    elif key == "yhi":
        s.y_hi = parse_bound(value)
    elif key == "ulo":
        s.u_lo = parse_bound(value)
    elif key == "uhi":
        s.u_hi = parse_bound(value)
    elif key == "delta":
        a.delta = _parse_double(key, value)
    elif key == "rho":
        a.rho = _parse_double(key, value)
    elif key == "tol":
        a.tol_primal = _parse_double(key, value)
    elif key == "max_outer":
        a.max_outer = _parse_int(key, value)
    elif key == "max_inner":
        a.max_inner = _parse_int(key, value)
    elif key == "inner_tol_floor":
        a.inner_tol_floor = _parse_double(key, value)
    elif key == "inner_tol_factor":
        a.inner_tol_factor = _parse_double(key, value)
    elif key == "warm_start":
        a.warm_start = _parse_flag(key, value)
    elif key == "out":
        cfg.out_dir = value
    elif key == "format":
        if value not in ("csv", "plain"):
            raise ConfigError(f"config key 'format' expects csv or plain, got '{value}'")
        cfg.format = value
    elif key == "delta_sweep":
        cfg.delta_sweep = _parse_list(key, value, _parse_double)
    elif key == "n_sweep":
        cfg.n_sweep = _parse_list(key, value, _parse_int)
    elif key == "alpha_sweep":
        cfg.alpha_sweep = _parse_list(key, value, _parse_double)
    elif key == "seed":
        cfg.seed = _parse_int(key, value) & 0xFFFFFFFF
    elif key == "dump":
        cfg.dump_solution = _parse_flag(key, value)
    elif key == "workers":
        cfg.workers = _parse_int(key, value)
    else:
        raise ConfigError(f"unknown config key '{key}'; valid keys: " + " ".join(CONFIG_KEYS))


def parse_config_file(path: str, cfg: RunConfig) -> None:
    """config.cpp:123-138"""
    try:
        fh = open(path)
    except OSError:
        raise ConfigError(f"cannot open config file '{path}'") from None
    with fh:
        for lineno, line in enumerate(fh, 1):
            line = line.rstrip("\n")
            if "#" in line:
                line = line[:line.index("#")]
            line = line.strip(" \t\r\n")
            if not line:
                continue
            if "=" not in line:
                raise ConfigError(f"config line {lineno}: expected key = value")
            k, v = line.split("=", 1)
            apply_config_entry(k.strip(" \t\r\n"), v.strip(" \t\r\n"), cfg)


# ------------------------------------------------------------------ problem
def grid_h(n: int) -> float:
    """Grid(n): h_x = h_t = 1/(n+1) (problem.cpp:22-24)."""
    if n < 1:
        raise ConfigError("Grid: n must be >= 1")
    return 1.0 / (n + 1)


def scaling_psi(spec: ProblemSpec) -> float:
    """scaling(spec, grid).psi (problem.cpp:26-33)."""
    spec.validate()
    h = grid_h(spec.n)
    return min(h ** spec.alpha, min(h ** spec.beta1, h ** spec.beta2))


def desired_state_at(x1, x2, t):
    """problem.cpp:47-49"""
    return 10.0 * np.cos(10.0 * x1) * np.sin(x1 * x2) * (1.0 - np.exp(-5.0 * t))


def desired_state(n: int) -> np.ndarray:
    """problem.cpp:51-58: layout (t, x1, x2), coordinates (i+1) h."""
    c = (np.arange(n) + 1.0) * grid_h(n)
    T, X1, X2 = np.meshgrid(c, c, c, indexing="ij")
    return desired_state_at(X1, X2, T).ravel()


def l2_misfit(y: np.ndarray, n: int) -> float:
    """problem.cpp:70-83 (interior rule sqrt(h^3) ||y - ybar||_2)."""
    h = grid_h(n)
    d = np.asarray(y, dtype=np.float64) - desired_state(n)
    return math.sqrt(float(np.dot(d, d)) * h * h * h)


def solve_spec(spec: ProblemSpec, admm: AdmmSettings, ctx=None, callback=None, keep_state=False) -> dict:
    """fdeopt::solve(spec, cfg) (admm.cpp:279-324) on the B200 path.  Returns
    the SolveResult fields the front end reports plus y, u and history."""
    import time

    from .api import (AdmmConfig, AdmmDriver, ConstraintOperator, assemble_precond, build_caputo,
                      build_riesz, solve)
    t0 = time.perf_counter()
    spec.validate()
    admm.validate()
    n, h = spec.n, grid_h(spec.n)
    psi = scaling_psi(spec)
    op = ConstraintOperator(build_caputo(spec.alpha, n, h), build_riesz(spec.beta1, n, h),
                            build_riesz(spec.beta2, n, h), psi, ctx=ctx)
    pc = assemble_precond(op, admm.rho, admm.delta, spec.gamma)
    cfg = AdmmConfig(delta=admm.delta, rho=admm.rho, tol_primal=admm.tol_primal, max_outer=admm.max_outer,
                     inner_tol_floor=admm.inner_tol_floor, inner_tol_factor=admm.inner_tol_factor,
                     max_inner=admm.max_inner, warm_start=admm.warm_start, fixed_krylov_tol=0.0)
    drv = AdmmDriver(op, pc, spec.gamma, cfg, y_lo=spec.y_lo, y_hi=spec.y_hi, u_lo=spec.u_lo,
                     u_hi=spec.u_hi, ybar=desired_state(n))
    res = solve(drv, callback)
    y = drv.get("y")
    u = drv.get("v") / psi
    res.update(y=y, u=u, misfit=l2_misfit(y, n), wall_seconds=time.perf_counter() - t0)
    if keep_state:  # the rest of SolveResult's state (admm.hpp:45-53)
        res.update({k: drv.get(k) for k in ("p", "w_y", "w_v", "z_y", "z_v")})
    return res
