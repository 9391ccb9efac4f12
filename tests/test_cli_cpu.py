"""CLI + bench harness, host side (no GPU): the reference's CLI/bench contract
(pkg/tests/test_cli.py, pkg/tests/test_bench.py) for everything that does
not launch a kernel, and the bench rendering pinned to the reference's own
output (tests/golden/cli_reference.json, tools/make_goldens.py cli)."""
import json
import subprocess
import sys
import time

import pytest

import paper_1701_03512_b200 as bp
from paper_1701_03512_b200 import BENCH_CSV_HEADER, BenchRecord, records_to_csv, records_to_tables, run_bench
from paper_1701_03512_b200.cli import main
from conftest import ROOT, gpu_available, load_golden

DESK = ["--payoff", "asian-put", "--S0", "20", "--K", "100", "--q", "0.06", "--sigma", "3.0", "--T", "1"]


def run_cli(capsys, *argv):
    code = main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


# --- bench harness (reference bench.py semantics) ---------------------------
def test_single_cell_is_its_own_baseline():
    (rec,) = run_bench([(10, 1)], lambda n, m: time.sleep(0.005), repetitions=1)
    assert (rec.speedup, rec.efficiency, rec.baseline_m) == (1.0, 1.0, 1)
    assert rec.wall_seconds > 0


def test_linear_synthetic_scaling_and_baseline_above_one():
    recs = run_bench([(8, m) for m in (1, 2, 4)], lambda n, m: time.sleep(0.08 / m), repetitions=3)
    for r in recs:
        assert r.efficiency == pytest.approx(1.0, abs=0.15)
    recs = run_bench([(8, m) for m in (2, 4)], lambda n, m: time.sleep(0.08 / m), repetitions=3)
    assert all(r.baseline_m == 2 for r in recs)
    assert recs[0].speedup == 2.0 and recs[0].efficiency == 1.0


def test_speedup_identity_exact():
    recs = run_bench([(5, 1), (5, 2)], lambda n, m: time.sleep(0.01), repetitions=1)
    for r in recs:
        assert r.speedup * r.wall_seconds == pytest.approx(recs[0].wall_seconds * recs[0].baseline_m, rel=1e-12)
        assert r.efficiency == r.speedup / r.m


@pytest.mark.parametrize("grid,reps", [([(8, 4), (8, 2)], 3), ([(8, 1), (10, 1), (8, 2)], 3), ([], 3),
                                       ([(8, 1)], 0), ([(8, 1)], True), ([(8, 2), (8, 2)], 3)])
def test_grid_validation(grid, reps):
    with pytest.raises(bp.InvalidInput):
        run_bench(grid, lambda n, m: None, repetitions=reps)


def test_rendering_matches_reference_bytes():
    g = load_golden("cli_reference.json")["bench_format"]
    recs = [BenchRecord(**r) for r in g["records"]]
    assert records_to_csv(recs) == g["csv"]
    assert records_to_tables(recs) == g["tables"]
    assert g["csv"].split("\n")[0] == BENCH_CSV_HEADER


# --- CLI usage errors and host-only methods ---------------------------------
@pytest.mark.parametrize("argv,needle", [
    (["price", "--method", "exact", "--N", "30", *DESK], "force-large"),
    (["price", "--method", "mc", "--N", "12", *DESK], "--samples"),
    (["price", "--method", "mc", "--N", "12", "--samples", "0", *DESK], "--samples"),
    (["price", "--method", "mc", "--N", "12", "--samples", "64", "--seed", "-1", *DESK], "seed"),
    (["price", "--method", "pmc", "--N", "12", "--samples", "64", "--workers", "0", *DESK], "--workers"),
    (["study", "--table", "mc-convergence", "--N", "10", *DESK], "--R-list"),
    (["study", "--table", "pmc-variance", "--N", "10", "--M-list", "2", *DESK], "--samples"),
    (["bench", "--N-list", "10", "--M-list", "4,2", *DESK], "ascending"),
    (["bench", "--N-list", "30", "--M-list", "1", *DESK], "force-large"),
    (["bench", "--N-list", "10", "--M-list", "1,x", *DESK], ""),
    (["price", "--method", "mc", "--payoff", "digital", "--S0", "1", "--K", "1", "--q", "0", "--sigma", ".1",
      "--T", "1", "--N", "4", "--samples", "8"], ""),
])
def test_usage_errors_exit_two(capsys, argv, needle):
    code, _, err = run_cli(capsys, *argv)
    assert code == 2
    assert needle in err


def test_domain_errors_exit_three(capsys):
    base = ["price", "--method", "exact", "--payoff", "euro-put", "--S0", "4", "--K", "5", "--q", "0",
            "--sigma", "0.3", "--T", "1"]
    code, _, err = run_cli(capsys, *base, "--N", "2", "--probs", "0.5,1.5")
    assert code == 3 and "(0, 1)" in err
    code, _, _ = run_cli(capsys, *base, "--N", "3", "--probs", "0.5,0.5")
    assert code == 3
    code, _, _ = run_cli(capsys, *base, "--N", "2", "--override-u", "0.9")
    assert code == 3


def test_leaf_method_is_host_side_and_matches_reference(capsys):
    # value_leaf_formula is O(N) host arithmetic (reference exact.py:136-157)
    for case in load_golden("cli_reference.json")["price"]:
        if case["report"]["method"] != "leaf":
            continue
        code, out, _ = run_cli(capsys, *case["argv"])
        assert code == 0
        rep = json.loads(out)
        want = case["report"]
        assert rep["value"] == pytest.approx(want["value"], rel=1e-12)
        assert {k: rep[k] for k in want if k != "value"} == {k: v for k, v in want.items() if k != "value"}


def test_help_hides_overrides(capsys):
    assert run_cli(capsys, "--help")[0] == 0
    code, out, _ = run_cli(capsys, "price", "--help")
    assert code == 0 and "--override-u" not in out and "--devices" in out


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_engine_methods_fail_loudly_without_gpu(capsys):
    code, _, err = run_cli(capsys, "price", "--method", "exact", "--N", "8", *DESK)
    assert code == 3 and "error" in err


def test_module_entry_point_leaf():
    proc = subprocess.run([sys.executable, "-m", "paper_1701_03512_b200", "price", "--method", "leaf", "--payoff",
                           "euro-put", "--S0", "4", "--K", "5", "--q", "0", "--sigma", "0.3", "--T", "1", "--N", "2",
                           "--format", "csv"], capture_output=True, text=True, cwd=ROOT)
    assert proc.returncode == 0, proc.stderr
    header, row = proc.stdout.strip().split("\n")
    assert header.split(",")[:2] == ["method", "payoff"] and row.startswith("leaf,euro-put")
