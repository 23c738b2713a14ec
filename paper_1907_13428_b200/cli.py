"""Command-line front end of the reference on the B200 path (f3).

    python -m paper_1907_13428_b200.cli solve  [--config F] [--n N] [--alpha A] ... [--out DIR] [--dump]
    python -m paper_1907_13428_b200.cli sweep  [same flags; n_sweep / alpha_sweep / delta_sweep lists]
    python -m paper_1907_13428_b200.cli validate [--cap 4] [--perturb 0] [--seed 1]
    python -m paper_1907_13428_b200.cli bench  [--n 16 32] [--reps 5]

A clone of proj/tools/fdeopt_main.cpp's `solve`, `sweep`, `validate` and
`bench` subcommands: the same flags, config-file keys (spec.py), precedence (file,
then flags, then $FDEOPT_OUT_DIR for the output directory), stdout summary
rows, output files (solve_summary.csv, solve_iterations.csv, y.bin / u.bin +
manifest.txt, sweep_summary.csv; formats in io.py) and exit codes (0 ok,
1 usage or solver failure, 2 iteration cap).  The solves run the reference's
own experiment (Caputo time factor, Riesz space factors, its desired state
and dynamic inner tolerance; spec.solve_spec) on the GPU; `validate` runs
the reference's dense-oracle suite (validation.py) against the B200 path
(exit 3 on a failed check).  `diagnose` (symbol / Wiener / clustering
diagnostics) is outside the hot path and not cloned.

sweep: points run one after another on this process's GPU; launched under
torchrun (one rank per GPU) the points are sharded round-robin over the
ranks (replicas.shard) and rank 0 prints and writes every row in point
order.  `--workers` is accepted for compatibility.
"""
from __future__ import annotations

import argparse
import math
import os
import sys
import time

from . import io as fio
from .spec import ConfigError, RunConfig, parse_bound, parse_config_file, solve_spec

EXIT_OK, EXIT_USAGE, EXIT_ITERCAP, EXIT_VALIDATION = 0, 1, 2, 3  # fdeopt_main.cpp:28-31


def _common_flags(p: argparse.ArgumentParser) -> None:
    """fdeopt_main.cpp:44-64 (None = not given)."""
    p.add_argument("--config", help="config file (key = value lines, # comments)")
    p.add_argument("--out", help="output directory (default: $FDEOPT_OUT_DIR)")
    p.add_argument("--n", type=int)
    for k in ("alpha", "beta1", "beta2", "gamma", "delta", "rho", "tol"):
        p.add_argument(f"--{k}", type=float)
    for k in ("ylo", "yhi", "ulo", "uhi"):
        p.add_argument(f"--{k}", help="bound (number or inf)")
    p.add_argument("--max-outer", type=int, dest="max_outer")
    p.add_argument("--workers", type=int)
    p.add_argument("--seed", type=int)
    p.add_argument("--dump", action="store_true", default=None)


def resolve_config(args) -> RunConfig:
    """fdeopt_main.cpp:66-93: file, then explicitly given flags, then env."""
    cfg = RunConfig()
    if args.config:
        parse_config_file(args.config, cfg)
    s, a = cfg.spec, cfg.admm
    if args.n is not None:
        s.n = args.n
    for k in ("alpha", "beta1", "beta2", "gamma"):
        if getattr(args, k) is not None:
            setattr(s, k, getattr(args, k))
    if args.delta is not None:
        a.delta = args.delta
    if args.rho is not None:
        a.rho = args.rho
    for flag, attr in (("ylo", "y_lo"), ("yhi", "y_hi"), ("ulo", "u_lo"), ("uhi", "u_hi")):
        if getattr(args, flag) is not None:
            setattr(s, attr, parse_bound(getattr(args, flag)))
    if args.tol is not None:
        a.tol_primal = args.tol
    if args.max_outer is not None:
        a.max_outer = args.max_outer
    if args.workers is not None:
        cfg.workers = args.workers
    if args.seed is not None:
        cfg.seed = args.seed & 0xFFFFFFFF
    if args.dump is not None:
        cfg.dump_solution = bool(args.dump)
    if args.out is not None:
        cfg.out_dir = args.out
    if not cfg.out_dir:
        cfg.out_dir = os.environ.get("FDEOPT_OUT_DIR", "")
    s.validate()
    a.validate()
    return cfg


def _row_text(cfg: RunConfig, row: fio.SummaryRow) -> str:
    return fio.summary_plain_row(row) if cfg.format == "plain" else fio.summary_csv_row(row)


def _write_summary_file(cfg: RunConfig, rows, name: str) -> None:
    """fdeopt_main.cpp:99-106"""
    if not cfg.out_dir:
        return
    os.makedirs(cfg.out_dir, exist_ok=True)
    with open(os.path.join(cfg.out_dir, name), "w") as fh:
        fh.write(fio.SUMMARY_HEADER + "\n")
        for r in rows:
            fh.write(fio.summary_csv_row(r) + "\n")


def _solver_failure(e: Exception) -> bool:
    from ._native import FdgError
    return isinstance(e, (FdgError, RuntimeError)) and not isinstance(e, ValueError)


def cmd_solve(args) -> int:
    """fdeopt_main.cpp:108-131"""
    cfg = resolve_config(args)
    try:
        result = solve_spec(cfg.spec, cfg.admm)
    except Exception as e:  # noqa: BLE001
        if not _solver_failure(e):
            raise
        print(f"solver failure: {e}", file=sys.stderr)
        return EXIT_USAGE
    row = fio.make_summary_row(cfg, cfg.admm.delta, result)
    if cfg.format == "csv":
        print(fio.SUMMARY_HEADER)
    print(_row_text(cfg, row), flush=True)
    if cfg.out_dir:
        _write_summary_file(cfg, [row], "solve_summary.csv")
        with open(os.path.join(cfg.out_dir, "solve_iterations.csv"), "w") as fh:
            fio.write_iteration_log(fh, result["history"])
        if cfg.dump_solution:
            d = cfg.out_dir
            fio.dump_solution(os.path.join(d, "y.bin"), cfg.spec.n, 0, result["y"])
            fio.dump_solution(os.path.join(d, "u.bin"), cfg.spec.n, 1, result["u"])
            fio.write_dump_manifest(os.path.join(d, "manifest.txt"), cfg.spec.n, [("y.bin", 0), ("u.bin", 1)])
    return EXIT_OK if result["status"] == "converged" else EXIT_ITERCAP


def sweep_points(cfg: RunConfig):
    """fdeopt_main.cpp:133-156: n x alpha x delta in that nesting order."""
    ns = cfg.n_sweep or [cfg.spec.n]
    alphas = cfg.alpha_sweep or [cfg.spec.alpha]
    deltas = cfg.delta_sweep or [cfg.admm.delta]
    pts = []
    for n in ns:
        for al in alphas:
            for de in deltas:
                p = cfg.copy()
                p.spec.n, p.spec.alpha, p.admm.delta = n, al, de
                pts.append(p)
    return pts


def _run_point(p: RunConfig, ctx=None):
    """fdeopt_main.cpp:159-175: (row, code); any failure -> a 'failed' row.
    ctx: the rank's device context (None: the default context, device 0)."""
    try:
        res = solve_spec(p.spec, p.admm, ctx=ctx)
        return fio.make_summary_row(p, p.admm.delta, res), (EXIT_OK if res["status"] == "converged" else EXIT_ITERCAP)
    except Exception:  # noqa: BLE001
        return fio.make_summary_row(p, p.admm.delta, {"status": "failed"}), EXIT_USAGE


def _rank_context(local: int):
    """The device context of this rank's solves (GPU LOCAL_RANK), or None
    without CUDA (the CPU gloo tests stub the solve)."""
    import torch
    if not torch.cuda.is_available():
        return None
    torch.cuda.set_device(local)
    from .api import Context
    return Context(local)


def cmd_sweep(args) -> int:
    """fdeopt_main.cpp:133-195"""
    cfg = resolve_config(args)
    if not (cfg.n_sweep or cfg.alpha_sweep or cfg.delta_sweep):
        print("sweep: no sweep list given (set n_sweep, alpha_sweep, or delta_sweep)", file=sys.stderr)
        return EXIT_USAGE
    pts = sweep_points(cfg)
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch
        import torch.distributed as dist
        from .replicas import gather_records, shard
        local = int(os.environ.get("LOCAL_RANK", "0"))
        ctx = _rank_context(local)  # every point of this rank solves on its own GPU
        own_group = not dist.is_initialized()
        if own_group:
            dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
        mine = shard(list(enumerate(pts)), rank, world)
        done = [(i, *_run_point(p, ctx)) for i, p in mine]
        allrec = gather_records([(i, vars(r), c) for i, r, c in done], dist)
        if own_group:
            dist.destroy_process_group()
        allrec.sort(key=lambda t: t[0])
        rows = [fio.SummaryRow(**r) for _, r, _ in allrec]
        codes = [c for _, _, c in allrec]
        if rank != 0:
            return EXIT_OK
    else:
        out = [_run_point(p) for p in pts]
        rows, codes = [r for r, _ in out], [c for _, c in out]
    if cfg.format == "csv":
        print(fio.SUMMARY_HEADER)
    for r in rows:
        print(_row_text(cfg, r))
    sys.stdout.flush()
    _write_summary_file(cfg, rows, "sweep_summary.csv")
    if all(c == EXIT_USAGE for c in codes):
        return EXIT_USAGE
    if any(c == EXIT_ITERCAP for c in codes):
        return EXIT_ITERCAP
    return EXIT_OK


def cmd_bench(sizes, reps: int) -> int:
    """fdeopt_main.cpp:261-293: best-of-reps wall time of one operator apply
    and one preconditioner solve on the reference default spec at each n
    (x_i = sin(0.37 i)), here device-resident with a device synchronize
    inside the timed call, and the process's peak RSS."""
    import numpy as np
    import torch

    from .api import Context, ConstraintOperator, assemble_precond, build_caputo, build_riesz
    from .spec import ProblemSpec, grid_h, scaling_psi
    print("n,N,apply_b_seconds,precond_solve_seconds,peak_rss_kb")
    ctx = Context(torch.cuda.current_device())
    for n in sizes:
        spec = ProblemSpec(n=n)
        h = grid_h(n)
        op = ConstraintOperator(build_caputo(spec.alpha, n, h), build_riesz(spec.beta1, n, h),
                                build_riesz(spec.beta2, n, h), scaling_psi(spec), ctx=ctx)
        pc = assemble_precond(op, 1.618, 0.4, spec.gamma)
        x = torch.tensor(np.sin(0.37 * np.arange(op.size)), dtype=torch.float64, device="cuda")
        out = torch.empty_like(x)
        torch.cuda.synchronize()

        def best(fn):
            b = math.inf
            for _ in range(reps):
                t0 = time.perf_counter()
                fn()
                ctx.synchronize()
                b = min(b, time.perf_counter() - t0)
            return b
        t_apply = best(lambda: op.apply_dev(x, out, False))
        t_solve = best(lambda: pc.solve_dev(x, out))
        print(f"{n},{op.size},{fio.fmt_g(t_apply)},{fio.fmt_g(t_solve)},{fio.fmt_g(fio.peak_rss_kb())}", flush=True)
    return EXIT_OK


def cmd_validate(cap: int, perturb: float, seed: int) -> int:
    """fdeopt_main.cpp:197-208: the dense-oracle equivalence suite
    (validation.py) against the B200 path; exit 3 on any failed check."""
    from .validation import B200Backend, format_report, run_validation
    results = run_validation(B200Backend(), cap, perturb, seed if seed else 1)
    print(format_report(results), flush=True)
    return EXIT_OK if all(r.passed() for r in results) else EXIT_VALIDATION


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="fdeopt-b200", description=(
        "matrix-free ADMM solver for box-constrained optimization governed by a time-dependent 2D "
        "fractional diffusion equation (B200 path)"))
    sub = ap.add_subparsers(dest="cmd", required=True)
    p_solve = sub.add_parser("solve", help="run a single solve and report a summary row")
    _common_flags(p_solve)
    p_sweep = sub.add_parser("sweep", help="run a sweep over n/alpha/delta lists")
    _common_flags(p_sweep)
    p_val = sub.add_parser("validate", help="run the dense-oracle equivalence suite")
    p_val.add_argument("--cap", type=int, default=4, choices=range(1, 7), metavar="[1-6]",
                       help="dense size cap (<= 6)")
    p_val.add_argument("--perturb", type=float, default=0.0,
                       help="fault-injection hook: perturb a discretization coefficient")
    p_val.add_argument("--seed", type=int, default=1, help="random seed")
    p_bench = sub.add_parser("bench", help="time apply/precond kernels, report peak RSS")
    p_bench.add_argument("--n", type=int, nargs="+", default=[16, 32])
    p_bench.add_argument("--reps", type=int, default=5)
    # bound values such as "-inf" after --ylo/--yhi/--ulo/--uhi are values,
    # not options (argparse would read them as flags)
    argv = list(sys.argv[1:] if argv is None else argv)
    for i in range(len(argv) - 1):
        if argv[i] in ("--ylo", "--yhi", "--ulo", "--uhi") and argv[i + 1].startswith("-"):
            argv[i], argv[i + 1] = f"{argv[i]}={argv[i + 1]}", ""
    argv = [a for a in argv if a != ""]
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:  # CLI11 parse errors -> usage exit code
        return EXIT_USAGE if e.code else EXIT_OK
    try:
        if args.cmd == "solve":
            return cmd_solve(args)
        if args.cmd == "sweep":
            return cmd_sweep(args)
        if args.cmd == "validate":
            return cmd_validate(args.cap, args.perturb, args.seed)
        return cmd_bench(args.n, args.reps)
    except (ConfigError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
