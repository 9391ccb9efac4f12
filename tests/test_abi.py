"""The C-ABI library loads and exports every symbol include/*.h declares
(CPU only: no compute calls)."""
import glob
import os
import re

import pytest

from conftest import ROOT


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        syms |= set(re.findall(r"\b(bp_[a-z0-9_]+)\s*\(", text))
    return syms


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert {"bp_exact", "bp_exact_superblocks", "bp_combine_superblocks", "bp_exact_batch", "bp_mc_strata",
            "bp_mc_shared", "bp_last_error"} <= syms


def test_library_exports_every_declared_symbol():
    from paper_1701_03512_b200 import _native
    if not _native.available():
        pytest.skip("engine not built")
    L = _native.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert set(_native.EXPORTED) == declared_symbols()
    assert L.bp_abi_version() == 1


def test_host_side_abi_functions_without_gpu():
    """bp_philox4x32_10 and bp_combine_superblocks are host code: callable here."""
    import ctypes
    import numpy as np
    from paper_1701_03512_b200 import _native
    if not _native.available():
        pytest.skip("engine not built")
    L = _native.lib()
    out = (ctypes.c_uint32 * 4)()
    L.bp_philox4x32_10((ctypes.c_uint32 * 4)(0, 0, 0, 0), (ctypes.c_uint32 * 2)(0, 0), out)
    assert list(out) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    parts = np.zeros((8, 6, 2))
    parts[:, 4, 0] = np.arange(8) * 0.1
    vals = np.zeros(6)
    assert L.bp_combine_superblocks(_native.dptr(parts), 8, 1 << 4, _native.dptr(vals)) == 0
    assert vals[4] == pytest.approx(2.8)
    # no device: engine entry points report it through the status code
    if _native.device_count() == 0:
        t, keep = _native.make_tree(4, 1.0, 1.0, 1.1, 0.9, 1.0, 0.5)
        res = _native.BpExactResult()
        rc = L.bp_exact(ctypes.byref(t), 1 << 4, 0, 0, None, ctypes.byref(res))
        assert rc == 101


def test_plain_c_client_builds_against_header_and_library():
    """examples/bp_price.c compiles and links against include/binpaths_b200.h
    and the built .so alone (runs on the GPU box, tests/test_c_client_gpu.py)."""
    import os
    from paper_1701_03512_b200 import build as b
    exe = b.build_example()
    assert os.access(exe, os.X_OK)
