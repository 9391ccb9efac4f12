"""The C ABI from plain C (examples/bp_price.c, built by build()): BASELINE
configs[0] against the reference golden, leaf bookkeeping, and the status-code
error path -- no Python between the caller and the engine."""
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_c_client_prices_config1_and_reports_errors():
    from paper_1701_03512_b200 import build as b
    exe = b.build_example()
    proc = subprocess.run([exe, "20"], capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert proc.returncode == 0, proc.stdout + proc.stderr
    assert "asian-call=6.02900791310063" in proc.stdout
    assert f"status {2}" in proc.stdout  # BP_E_PROBABILITY


def test_c_client_bookkeeping_large_N():
    from paper_1701_03512_b200 import build as b
    proc = subprocess.run([b.build_example(), "30"], capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert proc.returncode == 0, proc.stdout + proc.stderr
    assert "leaves=1073741824" in proc.stdout
