"""Result and wire formats of the reference (f2), byte-compatible.

Restates io.hpp / io.cpp (proj/include/fdeopt/io.hpp, proj/src/io.cpp):
  * fmt_g                       -- "%.12g" (io.cpp:9-13)
  * SUMMARY_HEADER, SummaryRow, make_summary_row, summary_csv_row,
    summary_plain_row           -- io.cpp:15-55
  * write_iteration_log         -- io.cpp:57-64
  * dump_solution, read_dump_header, read_dump -- FDEOPTv1 raw dumps: 32-byte
    header (magic "FDEOPTv1" | u32 n | u32 field id | u64 count | 8 zero
    bytes) + little-endian float64 payload (io.cpp:66-112)
  * write_dump_manifest         -- io.cpp:114-124
  * peak_rss_kb                 -- io.cpp:126-136
Golden bytes from the reference's own io.cpp: tests/golden/io/ (made by
tests/golden/make_io_golden.sh); the C++ facade's copy of these formats is
include/fdeopt_b200_io.hpp.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

MAGIC = b"FDEOPTv1"
SUMMARY_HEADER = "n,N,alpha,beta1,beta2,gamma,delta,rho,E_l2,dual_inf,pcg_avg,admm_iters,wall_seconds,status"


def fmt_g(v: float) -> str:
    """snprintf("%.12g") (io.cpp:9-13); glibc spells non-finite values
    inf / -inf / nan / -nan."""
    v = float(v)
    if v != v:
        return "-nan" if struct.pack("<d", v)[7] & 0x80 else "nan"
    return "%.12g" % v


@dataclass
class SummaryRow:
    """io.hpp:16-24"""
    n: int
    total: int
    alpha: float
    beta1: float
    beta2: float
    gamma: float
    delta: float
    rho: float
    e_l2: float
    dual_inf: float
    pcg_avg: float
    admm_iters: int
    wall_seconds: float
    status: str


def make_summary_row(cfg, delta: float, result: dict) -> SummaryRow:
    """io.cpp:18-35 (result: the dict of spec.solve_spec or a failure stub)."""
    s = cfg.spec
    return SummaryRow(s.n, s.n * s.n * s.n, s.alpha, s.beta1, s.beta2, s.gamma, delta, cfg.admm.rho,
                      result.get("misfit", 0.0), result.get("dual_inf", 0.0), result.get("pcg_avg", 0.0),
                      int(result.get("iterations", 0)), result.get("wall_seconds", 0.0),
                      {"converged": "converged", "itercap": "itercap"}.get(result.get("status"), "failed"))


def summary_csv_row(r: SummaryRow) -> str:
    """io.cpp:37-44"""
    return ",".join([str(r.n), str(r.total), fmt_g(r.alpha), fmt_g(r.beta1), fmt_g(r.beta2), fmt_g(r.gamma),
                     fmt_g(r.delta), fmt_g(r.rho), fmt_g(r.e_l2), fmt_g(r.dual_inf), fmt_g(r.pcg_avg),
                     str(r.admm_iters), fmt_g(r.wall_seconds), r.status])


def summary_plain_row(r: SummaryRow) -> str:
    """io.cpp:46-55"""
    return (f"n={r.n} N={r.total} alpha={fmt_g(r.alpha)} beta1={fmt_g(r.beta1)} beta2={fmt_g(r.beta2)} "
            f"gamma={fmt_g(r.gamma)} delta={fmt_g(r.delta)} rho={fmt_g(r.rho)} E_l2={fmt_g(r.e_l2)} "
            f"dual_inf={fmt_g(r.dual_inf)} pcg_avg={fmt_g(r.pcg_avg)} admm_iters={r.admm_iters} "
            f"wall_seconds={fmt_g(r.wall_seconds)} status={r.status}")


def write_iteration_log(fh, history) -> None:
    """io.cpp:57-64; history: IterRecord-like objects (iter, r_eq, r_y, r_u,
    dual_inf, inner_iters, inner_tol)."""
    fh.write("iter,r_eq,r_y,r_u,dual_inf,inner_iters,inner_tol\n")
    for rec in history:
        fh.write(f"{int(rec.iter)},{fmt_g(rec.r_eq)},{fmt_g(rec.r_y)},{fmt_g(rec.r_u)},{fmt_g(rec.dual_inf)},"
                 f"{int(rec.inner_iters)},{fmt_g(rec.inner_tol)}\n")


def dump_solution(path: str, n: int, field_id: int, data) -> None:
    """io.cpp:70-84"""
    a = np.ascontiguousarray(data, dtype="<f8")
    try:
        fh = open(path, "wb")
    except OSError:
        raise RuntimeError(f"cannot write '{path}'") from None
    with fh:
        fh.write(MAGIC + struct.pack("<IIQ", n & 0xFFFFFFFF, field_id & 0xFFFFFFFF, a.size) + bytes(8))
        fh.write(a.tobytes())


@dataclass
class DumpHeader:
    """io.hpp:38-42"""
    n: int
    field_id: int
    count: int


def read_dump_header(path: str) -> DumpHeader:
    """io.cpp:86-98"""
    try:
        fh = open(path, "rb")
    except OSError:
        raise RuntimeError(f"cannot read '{path}'") from None
    with fh:
        head = fh.read(32)
    if len(head) != 32 or head[:8] != MAGIC:
        raise RuntimeError(f"'{path}' is not a solution dump")
    n, fid, count = struct.unpack("<IIQ", head[8:24])
    return DumpHeader(n, fid, count)


def read_dump(path: str):
    """io.cpp:100-112: (data, header)."""
    h = read_dump_header(path)
    with open(path, "rb") as fh:
        fh.seek(32)
        raw = fh.read(h.count * 8)
    if len(raw) != h.count * 8:
        raise RuntimeError(f"'{path}' truncated")
    return np.frombuffer(raw, dtype="<f8").astype(np.float64), h


def write_dump_manifest(path: str, n: int, fields) -> None:
    """io.cpp:114-124; fields: [(file, id), ...]"""
    try:
        fh = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot write '{path}'") from None
    with fh:
        fh.write("format: raw little-endian float64 arrays\n")
        fh.write("header: 32 bytes = magic FDEOPTv1 | u32 n | u32 field_id | u64 count | 8 zero bytes\n")
        fh.write(f"n: {n}\n")
        fh.write(f"N: {n * n * n}\n")
        fh.write("layout: lexicographic, time outermost, then x1, then x2\n")
        for file, fid in fields:
            fh.write(f"field {fid}: {file}\n")


def peak_rss_kb() -> float:
    """io.cpp:126-136 (VmHWM of /proc/self/status)."""
    try:
        with open("/proc/self/status") as fh:
            for line in fh:
                if line.startswith("VmHWM:"):
                    return float(line.split()[1])
    except OSError:
        pass
    return 0.0
