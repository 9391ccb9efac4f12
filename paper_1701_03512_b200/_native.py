"""ctypes binding of the C ABI (include/binpaths_b200.h).

Loads ``_lib/libbinpaths_b200.so`` built in-tree by ``__graft_entry__.build()``
(or ``python -m paper_1701_03512_b200.build``).  There is no fallback: when
the library or a GPU is missing every engine call raises.  Status codes map
one-to-one onto the reference exception classes (errors.py:4-41).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BINPATHS_LIB") or os.path.join(_HERE, "_lib", "libbinpaths_b200.so")
N_PAYOFFS = 6

FLAG_COUNT = 1
FLAG_GENERIC = 2
FLAG_NO_TIMING = 4
FLAG_THRESHOLD = 8

_STATUS = E.STATUS_CLASSES


class BpTree(ctypes.Structure):
    _fields_ = [
        ("n_steps", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("S0", ctypes.c_double),
        ("K", ctypes.c_double),
        ("u", ctypes.c_double),
        ("d", ctypes.c_double),
        ("disc", ctypes.c_double),
        ("up_probs", ctypes.c_void_p),  # const double* (host); set from ndarray.ctypes.data
    ]


class BpExactResult(ctypes.Structure):
    _fields_ = [
        ("value", ctypes.c_double * N_PAYOFFS),
        ("leaves", ctypes.c_uint64),
        ("code_sum", ctypes.c_uint64),
        ("hist", ctypes.c_uint64 * 64),
        ("kernel_ms", ctypes.c_double),
        ("engine", ctypes.c_int32),
        ("inner_bits", ctypes.c_int32),
        ("n_superblocks", ctypes.c_int32),
        ("n_devices", ctypes.c_int32),
    ]


# every symbol the header declares (tests check the .so exports all of them)
EXPORTED = (
    "bp_exact", "bp_exact_layout", "bp_exact_superblocks", "bp_combine_superblocks", "bp_exact_batch",
    "bp_mc_strata", "bp_mc_range", "bp_mc_shared", "bp_philox4x32_10", "bp_fp64_peak", "bp_device_count",
    "bp_abi_version", "bp_last_error", "bp_exact_plan_create", "bp_exact_plan_layout", "bp_exact_plan_enqueue",
    "bp_exact_plan_destroy",
)

_lib = None
_lock = threading.Lock()


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    """The loaded engine library; raises loudly when it was not built."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise E.DeviceError(
                        f"CUDA engine not built ({LIB_PATH} missing); run __graft_entry__.build()")
                L = ctypes.CDLL(LIB_PATH)
                _declare(L)
                _lib = L
    return _lib


def _declare(L):
    c_int, c_u32, c_u64, c_dbl = ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double
    P = ctypes.POINTER
    L.bp_exact.argtypes = [P(BpTree), c_u32, c_u32, c_int, P(c_int), P(BpExactResult)]
    L.bp_exact_layout.argtypes = [P(BpTree), c_u32, c_u32, P(c_int), P(c_int), P(c_int)]
    L.bp_exact_superblocks.argtypes = [P(BpTree), c_u32, c_u32, c_int, c_int, c_int, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p]
    L.bp_exact_plan_create.argtypes = [P(BpTree), c_u32, c_u32, P(ctypes.c_void_p)]
    L.bp_exact_plan_layout.argtypes = [ctypes.c_void_p, P(c_int), P(c_int), P(c_int)]
    L.bp_exact_plan_enqueue.argtypes = [ctypes.c_void_p, c_int, c_int, c_int, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p]
    L.bp_exact_plan_destroy.argtypes = [ctypes.c_void_p]
    L.bp_exact_plan_destroy.restype = None
    L.bp_combine_superblocks.argtypes = [P(c_dbl), c_int, c_u32, P(c_dbl)]
    L.bp_exact_batch.argtypes = [P(BpTree), c_int, c_u32, c_int, P(c_dbl), P(c_dbl)]
    L.bp_mc_strata.argtypes = [P(BpTree), c_u32, c_int, P(c_u64), c_u64, c_u32, c_u32, c_int, P(c_dbl),
                               P(c_dbl), P(c_dbl)]
    L.bp_mc_range.argtypes = [P(BpTree), c_u32, c_int, P(c_u64), P(c_u64), c_u64, c_u32, c_u32, c_int, P(c_dbl),
                              P(c_dbl), P(c_dbl)]
    L.bp_mc_shared.argtypes = [P(BpTree), c_u32, c_int, c_u64, P(c_dbl), c_u64, c_u32, c_u32, c_int, P(c_dbl),
                               P(c_dbl), P(c_dbl), P(c_dbl)]
    L.bp_philox4x32_10.argtypes = [P(ctypes.c_uint32), P(ctypes.c_uint32), P(ctypes.c_uint32)]
    L.bp_philox4x32_10.restype = None
    L.bp_fp64_peak.argtypes = [c_int, P(c_dbl), P(c_dbl)]
    L.bp_device_count.argtypes = []
    L.bp_abi_version.argtypes = []
    L.bp_last_error.argtypes = []
    L.bp_last_error.restype = ctypes.c_char_p
    for name in EXPORTED:
        fn = getattr(L, name)
        if name not in ("bp_philox4x32_10", "bp_last_error", "bp_exact_plan_destroy"):
            fn.restype = c_int


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().bp_last_error().decode(errors="replace")
        raise _STATUS.get(rc, E.PricingError)(msg or f"engine status {rc}")


def dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def u64ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def make_tree(N, S0, K, u, d, disc, probs) -> tuple:
    """(BpTree, keep-alive array).  probs: per-step up probabilities."""
    p = probs
    if not (isinstance(p, np.ndarray) and p.dtype == np.float64 and p.shape == (N,) and p.flags.c_contiguous):
        p = np.ascontiguousarray(np.broadcast_to(np.asarray(probs, dtype=np.float64), (N,)), dtype=np.float64)
    t = BpTree(int(N), 0, float(S0), float(K), float(u), float(d), float(disc), p.ctypes.data)
    return t, p


def device_count() -> int:
    return int(lib().bp_device_count())
