"""bench.py --gpus N launcher (CPU): N > 1 runs N torchrun ranks or fails
loudly; never a silent one-GPU measurement."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT
from paper_1701_03512_b200 import launch


def test_bench_gpus_2_without_devices_fails_loudly():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode != 0
    assert "needs 2 visible CUDA devices" in out.stderr


def test_world_size_mismatch_is_an_error(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "4")
    with pytest.raises(launch.LaunchError):
        launch.ensure_world(8, "bench.py", [])
    assert launch.ensure_world(4, "bench.py", []) is None


def test_single_rank_runs_in_process(monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert launch.ensure_world(1, "bench.py", []) is None


def test_torchrun_command_uses_loopback():
    cmd = launch.torchrun_cmd("bench.py", ["--gpus", "8"], 8, port=29512)
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29512" in cmd
    assert cmd[-3:] == ["bench.py", "--gpus", "8"]


@pytest.mark.parametrize("world", [2, 3])
def test_launcher_runs_exact_exchange_ranks(world, tmp_path, monkeypatch):
    """The launcher starts `world` ranks; each exchanges its super-block
    partials (64 canonical super-blocks; 22/21/21 at world 3) and all ranks
    combine to the same value, equal to the oracle's full enumeration."""
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    rc = launch.ensure_world(world, os.path.join(ROOT, "tests", "_launch_worker.py"), [str(tmp_path)],
                             need_devices=False)
    assert rc == 0
    res = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    assert sum(r["count"] for r in res) == 64
    assert all(r["values"] == res[0]["values"] for r in res)
    import oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _launch_worker as w
    full = oracle.exact(w.N, w.S0, w.K, w.U, 1 / w.U, w.P, w.DISC, w.KINDS)
    for k in full:
        assert res[0]["values"][k] == pytest.approx(full[k], rel=1e-13)
