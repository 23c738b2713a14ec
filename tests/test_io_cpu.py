"""Result / wire formats and the run configuration of the reference
(f2, f3) -- CPU only.

Golden files: the reference's own io.cpp output (tests/golden/io, made by
tests/golden/make_io_golden.sh).  Checked: the Python restatement
(paper_1907_13428_b200/io.py) and the C++ facade header
(include/fdeopt_b200_io.hpp, compiled here with g++) reproduce them byte for
byte; the config parser follows config.cpp (keys, lists, flags, errors); the
CLI resolves file / flag / environment precedence as fdeopt_main.cpp.
"""
import math
import os
import shutil
import subprocess

import numpy as np
import pytest

from paper_1907_13428_b200 import io as fio
from paper_1907_13428_b200.spec import (CONFIG_KEYS, AdmmSettings, ConfigError, ProblemSpec, RunConfig,
                                        apply_config_entry, desired_state, l2_misfit, parse_bound,
                                        parse_config_file)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "io")


def _read(name, mode="rb"):
    with open(os.path.join(GOLD, name), mode) as fh:
        return fh.read()


SUMMARY_ROWS = [
    fio.SummaryRow(12, 1728, 0.7, 1.3, 1.2999999999999998, 1e-4, 0.4, 1.618, 0.0123456789012345, 3.5e-17,
                   13.4615384615, 42, 1234.5678901234567, "converged"),
    fio.SummaryRow(8, 512, 0.5, 1.5, 1.5, 2.5e-300, 1e21, 1.0, math.inf, -math.inf, 0.0, 0, 0.1, "failed"),
]


class Rec:
    def __init__(self, k):
        self.iter, self.r_eq, self.r_y = k + 1, 0.1 / (k + 1), 1e-7 * (k + 2)
        self.r_u, self.dual_inf = 2.0 / 3.0 * k, 10.0 ** (-k) * math.pi
        self.inner_iters, self.inner_tol = 10 + k, 5e-6


def test_dump_bytes_match_reference(tmp_path):
    data, h = fio.read_dump(os.path.join(GOLD, "u.bin"))
    assert (h.n, h.field_id, h.count) == (3, 1, 27)
    assert np.isneginf(data[6]) and np.isposinf(data[5]) and math.copysign(1.0, data[3]) < 0
    out = tmp_path / "u.bin"
    fio.dump_solution(str(out), 3, 1, data)
    assert out.read_bytes() == _read("u.bin")
    fio.dump_solution(str(tmp_path / "e.bin"), 0, 0, np.zeros(0))
    assert (tmp_path / "e.bin").read_bytes() == _read("empty.bin")


def test_dump_errors(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"FDEOPTv2" + bytes(24))
    with pytest.raises(RuntimeError, match="is not a solution dump"):
        fio.read_dump(str(bad))
    tr = tmp_path / "tr.bin"
    tr.write_bytes(_read("u.bin")[:-8])
    with pytest.raises(RuntimeError, match="truncated"):
        fio.read_dump(str(tr))
    with pytest.raises(RuntimeError, match="cannot read"):
        fio.read_dump_header(str(tmp_path / "missing.bin"))


def test_text_formats_match_reference(tmp_path):
    csv = fio.SUMMARY_HEADER + "\n" + "".join(fio.summary_csv_row(r) + "\n" for r in SUMMARY_ROWS)
    assert csv == _read("summary.csv", "r")
    plain = "".join(fio.summary_plain_row(r) + "\n" for r in SUMMARY_ROWS)
    assert plain == _read("summary_plain.txt", "r")
    with open(tmp_path / "it.csv", "w") as fh:
        fio.write_iteration_log(fh, [Rec(k) for k in range(3)])
    assert (tmp_path / "it.csv").read_text() == _read("iterations.csv", "r")
    fio.write_dump_manifest(str(tmp_path / "m.txt"), 3, [("y.bin", 0), ("u.bin", 1)])
    assert (tmp_path / "m.txt").read_text() == _read("manifest.txt", "r")
    assert fio.fmt_g(float("nan")) == "nan" and fio.fmt_g(-float("nan")) == "-nan"


CPP = r'''
#include <cmath>
#include <fstream>
#include <limits>
#include "fdeopt_b200_io.hpp"
using namespace fdeopt::b200;
int main(int argc, char** argv) {
  const std::string d = argv[1], g = argv[2];
  DumpHeader h;
  std::vector<double> v = read_dump(g + "/u.bin", &h);
  dump_solution(d + "/u.bin", h.n, h.field_id, v);
  dump_solution(d + "/empty.bin", 0, 0, {});
  write_dump_manifest(d + "/manifest.txt", 3, {{"y.bin", 0}, {"u.bin", 1}});
  SummaryRow r{12, 1728, 0.7, 1.3, 1.2999999999999998, 1e-4, 0.4, 1.618, 0.0123456789012345,
               3.5e-17, 13.4615384615, 42, 1234.5678901234567, "converged"};
  SummaryRow f{8, 512, 0.5, 1.5, 1.5, 2.5e-300, 1e+21, 1.0, std::numeric_limits<double>::infinity(),
               -std::numeric_limits<double>::infinity(), 0.0, 0, 0.1, to_string(SolveStatus::failure)};
  std::ofstream csv(d + "/summary.csv");
  csv << kSummaryHeader << "\n" << summary_csv_row(r) << "\n" << summary_csv_row(f) << "\n";
  std::ofstream plain(d + "/summary_plain.txt");
  plain << summary_plain_row(r) << "\n" << summary_plain_row(f) << "\n";
  std::vector<IterRecord> hist;
  for (int k = 0; k < 3; ++k)
    hist.push_back(IterRecord{k + 1, 0.1 / (k + 1), 1e-7 * (k + 2), 2.0 / 3.0 * k, std::pow(10.0, -k) * M_PI,
                              10 + k, 5e-6});
  std::ofstream log(d + "/iterations.csv");
  write_iteration_log(log, hist);
  return peak_rss_kb() > 0.0 ? 0 : 1;
}
'''


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_cpp_facade_io_matches_reference(tmp_path):
    src = tmp_path / "io_check.cpp"
    src.write_text(CPP)
    exe = tmp_path / "io_check"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = tmp_path / "out"
    out.mkdir()
    subprocess.run([str(exe), str(out), GOLD], check=True)
    for name in ("u.bin", "empty.bin", "manifest.txt", "summary.csv", "summary_plain.txt", "iterations.csv"):
        assert (out / name).read_bytes() == _read(name), name


def test_config_file_and_entries(tmp_path):
    p = tmp_path / "run.cfg"
    p.write_text("# reference experiment\n n = 12   # grid\nalpha=0.5\nbeta1 = 1.4\nylo = -inf\nuhi = 2\n"
                 "delta_sweep = 0.1, 0.2,0.4\nn_sweep = 4,8\nwarm_start = yes\nformat = plain\n"
                 "dump = 1\nseed = 7\nmax_inner = 50\ninner_tol_floor = 1e-5\n\n")
    cfg = RunConfig()
    parse_config_file(str(p), cfg)
    s, a = cfg.spec, cfg.admm
    assert (s.n, s.alpha, s.beta1, s.beta2) == (12, 0.5, 1.4, 1.3)
    assert s.y_lo == -math.inf and s.u_hi == 2.0 and s.u_lo == -math.inf
    assert cfg.delta_sweep == [0.1, 0.2, 0.4] and cfg.n_sweep == [4, 8]
    assert a.warm_start and cfg.format == "plain" and cfg.dump_solution and cfg.seed == 7
    assert (a.max_inner, a.inner_tol_floor, a.delta, a.rho) == (50, 1e-5, 0.4, 1.618)
    assert len(CONFIG_KEYS) == 25


@pytest.mark.parametrize("key,value,msg", [
    ("n", "8.5", "config key 'n' expects an integer, got '8.5'"),
    ("alpha", "0.5x", "config key 'alpha' expects a number, got '0.5x'"),
    ("warm_start", "maybe", "config key 'warm_start' expects a boolean, got 'maybe'"),
    ("format", "json", "config key 'format' expects csv or plain, got 'json'"),
    ("n_sweep", " , ", "config key 'n_sweep' expects a nonempty list"),
    ("colour", "red", "unknown config key 'colour'; valid keys: alpha beta1"),
])
def test_config_errors(key, value, msg):
    with pytest.raises(ConfigError) as e:
        apply_config_entry(key, value, RunConfig())
    assert str(e.value).startswith(msg)


def test_config_file_errors(tmp_path):
    p = tmp_path / "bad.cfg"
    p.write_text("n = 4\njust words\n")
    with pytest.raises(ConfigError, match="config line 2: expected key = value"):
        parse_config_file(str(p), RunConfig())
    with pytest.raises(ConfigError, match="cannot open config file"):
        parse_config_file(str(tmp_path / "none.cfg"), RunConfig())


def test_spec_validation_and_bounds():
    assert parse_bound(" +inf ") == math.inf and parse_bound("-2.5") == -2.5
    for kw, msg in [({"alpha": 1.0}, "alpha must lie in (0, 1), got 1.000000"),
                    ({"beta2": 2.0}, "beta2 must lie in (1, 2), got 2.000000"),
                    ({"gamma": 0.0}, "gamma must be positive"), ({"n": 0}, "n must be >= 1"),
                    ({"y_lo": 1.0, "y_hi": 1.0}, "state bounds must satisfy y_lo < y_hi")]:
        with pytest.raises(ConfigError, match=msg.replace("(", r"\(").replace(")", r"\)")):
            ProblemSpec(**kw).validate()
    with pytest.raises(ConfigError, match="rho must lie"):
        AdmmSettings(rho=1.7).validate()
    with pytest.raises(ConfigError, match="iteration caps"):
        AdmmSettings(max_outer=0).validate()


def test_desired_state_and_misfit_match_reference(ref):
    n = 5
    want = np.zeros(n ** 3)
    ref.lib.ref_desired_state(n, want.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double)))
    assert np.array_equal(desired_state(n), want)
    y = want + 0.5
    assert abs(l2_misfit(y, n) - math.sqrt(0.25 * n ** 3 / (n + 1) ** 3)) < 1e-15


def test_cli_precedence(tmp_path, monkeypatch):
    from paper_1907_13428_b200 import cli
    p = tmp_path / "c.cfg"
    p.write_text("n = 6\ndelta = 0.3\nout = from_file\n")
    ap = __import__("argparse").ArgumentParser()
    cli._common_flags(ap)
    args = ap.parse_args(["--config", str(p), "--delta", "0.5", "--ulo=-inf", "--uhi", "3"])
    cfg = cli.resolve_config(args)
    assert (cfg.spec.n, cfg.admm.delta, cfg.out_dir, cfg.spec.u_hi) == (6, 0.5, "from_file", 3.0)
    monkeypatch.setenv("FDEOPT_OUT_DIR", str(tmp_path / "env"))
    args = ap.parse_args(["--n", "4"])
    assert cli.resolve_config(args).out_dir == str(tmp_path / "env")
    assert cli.main(["solve", "--rho", "2"]) == cli.EXIT_USAGE
    pts = cli.sweep_points(RunConfig(n_sweep=[4, 8], alpha_sweep=[0.3, 0.6], delta_sweep=[1.0]))
    assert [(q.spec.n, q.spec.alpha, q.admm.delta) for q in pts] == [(4, 0.3, 1.0), (4, 0.6, 1.0),
                                                                        (8, 0.3, 1.0), (8, 0.6, 1.0)]
