"""The reference's front end (fdeopt_main.cpp solve / sweep / bench) on the
B200 path (f3) against the unchanged reference's own
`fdeopt::solve` (oracle/_ref): the reference experiment (Caputo alpha = 0.7,
Riesz 1.3, its desired state, dynamic inner tolerance) end to end, with the
output files in the reference's formats."""
import csv
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rows(path):
    with open(path) as fh:
        return list(csv.DictReader(fh))


@pytest.mark.parametrize("n,extra", [(8, {}), (4, {"ulo": -0.5, "uhi": 0.4, "delta": 0.8}), (16, {}),
                                   (6, {"ulo": -0.5, "uhi": 0.4, "delta": 0.8}), (12, {})])
def test_cli_solve_matches_reference_solve(gpu_ctx, ref, tmp_path, capsys, n, extra):
    from paper_1907_13428_b200 import cli
    from paper_1907_13428_b200 import io as fio
    argv = ["solve", "--n", str(n), "--out", str(tmp_path), "--dump"]
    for k, v in extra.items():
        argv += [f"--{k}", str(v)]
    rc = cli.main(argv)
    want = ref.solve(n=n, u_lo=extra.get("ulo", -math.inf), u_hi=extra.get("uhi", math.inf),
                     delta=extra.get("delta", 0.4))
    cap = capsys.readouterr()
    out = cap.out.strip().splitlines()
    assert out and out[0] == fio.SUMMARY_HEADER, (rc, cap.err)
    assert rc == (0 if want["status"] == "converged" else 2)
    got = _rows(tmp_path / "solve_summary.csv")[0]
    assert got["status"] == want["status"]
    assert int(got["admm_iters"]) == want["iterations"]
    hist = _rows(tmp_path / "solve_iterations.csv")
    assert len(hist) == want["iterations"]
    inner = np.array([int(h["inner_iters"]) for h in hist])
    assert np.all(np.abs(inner - want["history"][:, 5]) <= 1)
    assert abs(float(got["pcg_avg"]) - want["pcg_avg"]) <= 1.0
    for k, w in (("E_l2", want["misfit"]), ("dual_inf", want["dual_inf"])):
        assert abs(float(got[k]) - w) <= 1e-6 * abs(w) + 1e-12, (k, got[k], w)
    y, hy = fio.read_dump(str(tmp_path / "y.bin"))
    u, hu = fio.read_dump(str(tmp_path / "u.bin"))
    assert (hy.n, hy.field_id, hy.count, hu.field_id) == (n, 0, n ** 3, 1)
    assert np.linalg.norm(y - want["y"]) <= 1e-6 * np.linalg.norm(want["y"])
    assert np.linalg.norm(u - want["u"]) <= 1e-6 * np.linalg.norm(want["u"])
    assert (tmp_path / "manifest.txt").read_text().splitlines()[2] == f"n: {n}"


def test_cli_sweep_and_itercap(gpu_ctx, tmp_path, capsys):
    from paper_1907_13428_b200 import cli
    cfg = tmp_path / "sweep.cfg"
    cfg.write_text("n = 4\ndelta_sweep = 0.4, 0.8\nformat = plain\n")
    rc = cli.main(["sweep", "--config", str(cfg), "--out", str(tmp_path)])
    lines = capsys.readouterr().out.strip().splitlines()
    assert rc == 0 and len(lines) == 2 and lines[0].startswith("n=4 N=64 ") and "delta=0.8 " in lines[1]
    rows = _rows(tmp_path / "sweep_summary.csv")
    assert [r["delta"] for r in rows] == ["0.4", "0.8"] and all(r["status"] == "converged" for r in rows)
    rc = cli.main(["solve", "--n", "4", "--max-outer", "2"])
    assert rc == 2 and capsys.readouterr().out.strip().splitlines()[1].endswith(",itercap")


def test_cli_bench(gpu_ctx, capsys):
    from paper_1907_13428_b200 import cli
    assert cli.main(["bench", "--n", "8", "16", "--reps", "2"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "n,N,apply_b_seconds,precond_solve_seconds,peak_rss_kb"
    assert [ln.split(",")[:2] for ln in lines[1:]] == [["8", "512"], ["16", "4096"]]
    assert all(float(ln.split(",")[2]) > 0 for ln in lines[1:])
