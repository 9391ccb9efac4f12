"""CLI wired to the GPU engine: the reference's CLI tests
(pkg/tests/test_cli.py) against this package's ``price`` / ``study`` /
``bench``, plus the exact-method reports pinned to the reference CLI's own
output (tests/golden/cli_reference.json)."""
import json
import subprocess
import sys

import pytest

from paper_1701_03512_b200.cli import REPORT_KEYS, STUDY_HEADER, main
from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu

DESK = ["--payoff", "asian-put", "--S0", "20", "--K", "100", "--q", "0.06", "--sigma", "3.0", "--T", "1"]


def run_cli(capsys, *argv):
    code = main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


def price(capsys, *argv):
    code, out, err = run_cli(capsys, "price", *argv)
    assert code == 0, err
    return json.loads(out)


def test_exact_reports_match_reference_cli():
    import contextlib
    import io
    g = load_golden("cli_reference.json")
    for case in g["price"]:
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            assert main(case["argv"]) == 0
        rep, want = json.loads(buf.getvalue()), case["report"]
        assert rep["value"] == pytest.approx(want["value"], rel=1e-12, abs=1e-14), case["argv"]
        for k, v in want.items():
            if k != "value":
                assert rep[k] == v, (k, case["argv"])


def test_hand_example_with_overrides(capsys):
    rep = price(capsys, "--method", "exact", "--payoff", "euro-put", "--S0", "4", "--K", "5", "--q", "0",
                "--sigma", "0.30", "--T", "1", "--N", "2", "--override-u", "2", "--override-p", "0.5")
    want = load_golden("cli_reference.json")["hand_example"]
    assert rep["value"] == pytest.approx(1.5, abs=1e-12)
    assert {k: rep[k] for k in want} == want


def test_report_key_order(capsys):
    rep = price(capsys, "--method", "mc", "--N", "12", "--samples", "64", *DESK)
    assert tuple(rep) == REPORT_KEYS
    assert rep["M"] == 1 and rep["R"] == 64 and rep["reps"] == 1
    rep = price(capsys, "--method", "mc", "--N", "12", "--samples", "64", "--reps", "5", *DESK)
    assert list(rep)[-1] == "empirical_variance" and rep["reps"] == 5


def test_pmc_single_worker_matches_mc_bitwise(capsys):
    mc = price(capsys, "--method", "mc", "--N", "12", "--samples", "1024", "--seed", "7", *DESK)
    pmc = price(capsys, "--method", "pmc", "--N", "12", "--samples", "1024", "--seed", "7", "--workers", "1", *DESK)
    for k in ("value", "variance", "std_error", "M", "R"):
        assert mc[k] == pmc[k]


def test_repeatable_and_eval_threads_invariant(capsys):
    runs = [price(capsys, "--method", "smc", "--N", "12", "--samples", "512", "--seed", "3", "--workers", "8", *DESK)
            for _ in range(3)]
    assert len({(r["value"], r["variance"]) for r in runs}) == 1
    runs = [price(capsys, "--method", "pmc", "--N", "12", "--samples", "512", "--seed", "3", "--workers", "8",
                  "--eval-threads", str(t), *DESK) for t in (1, 2, 4)]
    assert len({(r["value"], r["variance"]) for r in runs}) == 1


def test_gpu_payoffs_and_devices_flag(capsys):
    # the BASELINE config-1 tree through the CLI: Asian call, classic CRR via overrides
    import math
    u = math.exp(0.2 * math.sqrt(1 / 20))
    p = (math.exp(0.05 / 20) - 1 / u) / (u - 1 / u)
    rep = price(capsys, "--method", "exact", "--payoff", "asian-call", "--S0", "100", "--K", "100", "--q", "0.05",
                "--sigma", "0.2", "--T", "1", "--N", "20", "--override-u", repr(u), "--override-p", repr(p),
                "--devices", "0")
    g1 = load_golden("exact_config1.json")
    assert rep["value"] == pytest.approx(g1["asian_call"], rel=1e-12)


def test_mc_r_below_minimum_is_domain_error(capsys):
    code, _, _ = run_cli(capsys, "price", "--method", "mc", "--N", "12", "--samples", "1", *DESK)
    assert code == 3


def test_study_tables(capsys):
    common = ["--N", "10", "--seed", "3", "--reps", "5", *DESK]
    code, out_pmc, _ = run_cli(capsys, "study", "--table", "pmc-variance", "--M-list", "1", "--samples", "256",
                               *common)
    assert code == 0
    code, out_mc, _ = run_cli(capsys, "study", "--table", "mc-convergence", "--R-list", "256", *common)
    assert code == 0
    assert out_pmc.strip().split("\n")[1].split(",")[2:] == out_mc.strip().split("\n")[1].split(",")[2:]
    code, out, _ = run_cli(capsys, "study", "--table", "smc-vs-pmc", "--M-list", "2,4", "--samples", "128",
                           "--N", "10", "--reps", "3", *DESK)
    assert code == 0
    lines = out.strip().split("\n")
    assert lines[0] == STUDY_HEADER
    assert [ln.split(",")[0] for ln in lines[1:]] == ["pmc-equal", "smc", "pmc-equal", "smc"]


def test_bench_grid(capsys):
    code, out, _ = run_cli(capsys, "bench", "--N-list", "10", "--M-list", "1", "--reps", "1", *DESK)
    assert code == 0
    lines = out.strip().split("\n")
    assert lines[0].startswith("N,M,wall_seconds") and len(lines) == 2
    assert lines[1].split(",")[:2] == ["10", "1"] and float(lines[1].split(",")[3]) == 1.0
    code, out, _ = run_cli(capsys, "bench", "--N-list", "12,16", "--M-list", "1,2,4", "--reps", "2", *DESK)
    assert code == 0
    rows = out.strip().split("\n")[1:]
    assert len(rows) == 6 and all(float(r.split(",")[2]) > 0 for r in rows)
    code, out, _ = run_cli(capsys, "bench", "--N-list", "12", "--M-list", "1,2", "--reps", "1", "--format", "plain",
                           *DESK)
    assert code == 0 and "efficiency" in out and "N\\M" in out


def test_module_entry_point_exact():
    proc = subprocess.run([sys.executable, "-m", "paper_1701_03512_b200", "price", "--method", "exact", "--payoff",
                           "euro-put", "--S0", "4", "--K", "5", "--q", "0", "--sigma", "0.3", "--T", "1", "--N", "2"],
                          capture_output=True, text=True, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr
    assert json.loads(proc.stdout)["N"] == 2
