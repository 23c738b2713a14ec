"""The reference's dense-oracle equivalence suite (oracle.cpp:304-595) against
the B200 path, through the front end (`cli validate`, fdeopt_main.cpp:197-208):
every check within the reference's thresholds; the fault-injection hook makes
the unit-basis check fail with exit code 3."""
import pytest

pytestmark = pytest.mark.gpu


def test_cli_validate_passes(gpu_ctx, capsys):
    from paper_1907_13428_b200 import cli
    rc = cli.main(["validate", "--cap", "4", "--seed", "2"])
    out = capsys.readouterr().out
    rows = [ln.split() for ln in out.strip().splitlines()[1:]]
    assert rc == 0, out
    assert len(rows) == 10 and all(r[-1] == "PASS" for r in rows), out


def test_cli_validate_fault_injection(gpu_ctx, capsys):
    from paper_1907_13428_b200 import cli
    rc = cli.main(["validate", "--cap", "2", "--perturb", "1e-6"])
    out = capsys.readouterr().out
    res = {ln.split()[0]: ln.split()[-1] for ln in out.strip().splitlines()[1:]}
    assert rc == 3 and res["matvec_unit_basis"] == "FAIL", out
    assert all(v == "PASS" for k, v in res.items() if k != "matvec_unit_basis"), out
