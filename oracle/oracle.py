"""ctypes wrapper of the C oracle (test infrastructure only; see __init__)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "build", "libbp_oracle.so")

# kind name -> bit position, identical to include/binpaths_b200.h bp_payoff
KIND_BITS = {
    "euro-call": 0,
    "euro-put": 1,
    "asian-put": 2,
    "lookback-put": 3,
    "asian-call": 4,
    "float-lookback": 5,
}

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/bp_oracle.c into oracle/build/libbp_oracle.so."""
    src = os.path.join(_HERE, "bp_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_SO), exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-pthread", "-o", _SO, src, "-lm"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        d, i, u, u64 = ctypes.c_double, ctypes.c_int, ctypes.c_uint, ctypes.c_uint64
        pd = ctypes.POINTER(ctypes.c_double)
        pu64 = ctypes.POINTER(ctypes.c_uint64)
        pu32 = ctypes.POINTER(ctypes.c_uint32)
        L.orc_exact.argtypes = [i, d, d, d, d, pd, d, u, i, i, pd, pu64]
        L.orc_exact.restype = i
        L.orc_exact_range.argtypes = [i, d, d, d, d, pd, d, u, u64, u64, i, pd]
        L.orc_exact_range.restype = u64
        L.orc_philox4x32_10.argtypes = [pu32, pu32, pu32]
        L.orc_philox4x32_10.restype = None
        L.orc_mc_strata.argtypes = [i, d, d, d, d, pd, i, i, pu64, u64, ctypes.c_uint32, ctypes.c_uint32, pd, pd]
        L.orc_mc_strata.restype = i
        L.orc_mc_range.argtypes = [i, d, d, d, d, pd, i, i, pu64, pu64, u64, ctypes.c_uint32, ctypes.c_uint32, pd, pd]
        L.orc_mc_range.restype = i
        L.orc_mc_bits.argtypes = [i, i, pd, u64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                  ctypes.POINTER(ctypes.c_int)]
        L.orc_mc_bits.restype = None
        L.orc_mc_shared.argtypes = [i, d, d, d, d, pd, i, i, u64, pd, u64, ctypes.c_uint32, ctypes.c_uint32,
                                    pd, pd, pd]
        L.orc_mc_shared.restype = i
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _probs(N, p):
    arr = np.ascontiguousarray(np.broadcast_to(np.asarray(p, dtype=np.float64), (N,)), dtype=np.float64)
    return arr


def exact(N, S0, K, u, d, p, disc, kinds, workers=1, threads=None, with_hist=False):
    """value_exact_parallel restated; returns {kind: value} (+ hist)."""
    probs = _probs(N, p)
    mask = 0
    for k in kinds:
        mask |= 1 << KIND_BITS[k]
    vals = np.zeros(6)
    hist = np.zeros(N + 1, dtype=np.uint64) if with_hist else None
    th = threads or min(workers, os.cpu_count() or 1)
    rc = lib().orc_exact(N, S0, K, u, d, _dp(probs), disc, mask, workers, th, _dp(vals),
                         hist.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)) if with_hist else None)
    if rc != 0:
        raise AssertionError("oracle path accounting mismatch")
    out = {k: float(vals[KIND_BITS[k]]) for k in kinds}
    return (out, hist) if with_hist else out


def exact_range(N, S0, K, u, d, p, disc, kinds, lo, hi, threads=1):
    """Discounted partial sum over path codes [lo, hi) (bounded CPU sample)."""
    probs = _probs(N, p)
    mask = 0
    for k in kinds:
        mask |= 1 << KIND_BITS[k]
    vals = np.zeros(6)
    n = lib().orc_exact_range(N, S0, K, u, d, _dp(probs), disc, mask, lo, hi, threads, _dp(vals))
    return {k: float(vals[KIND_BITS[k]]) for k in kinds}, int(n)


def philox4x32_10(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return list(o)


def mc_strata(N, S0, K, u, d, probs, kind, r, draws, seed, rep0=0, n_reps=1):
    probs = _probs(N, probs)
    draws = np.ascontiguousarray(draws, dtype=np.uint64)
    M = 1 << r
    theta = np.zeros(n_reps * M)
    sse = np.zeros(n_reps * M)
    lib().orc_mc_strata(N, S0, K, u, d, _dp(probs), KIND_BITS[kind], r,
                        draws.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), seed, rep0, n_reps,
                        _dp(theta), _dp(sse))
    return theta.reshape(n_reps, M), sse.reshape(n_reps, M)


def mc_bits(N, r, probs, seed, stream=0, rep=0, draw=0):
    """Up/down bits of the N - r suffix steps of one draw (the sampler alone)."""
    probs = _probs(N, probs)
    up = (ctypes.c_int * max(N - r, 1))()
    lib().orc_mc_bits(N, r, _dp(probs), seed, stream, rep, draw, up)
    return np.array(list(up)[:N - r], dtype=bool)


def mc_range(N, S0, K, u, d, probs, kind, r, first, end, seed, rep0=0, n_reps=1):
    """Per-stratum (mean, M2) over draws [first[m], end[m]) (bp_mc_range)."""
    probs = _probs(N, probs)
    first = np.ascontiguousarray(first, dtype=np.uint64)
    end = np.ascontiguousarray(end, dtype=np.uint64)
    M = 1 << r
    mean = np.zeros(n_reps * M)
    m2 = np.zeros(n_reps * M)
    lib().orc_mc_range(N, S0, K, u, d, _dp(probs), KIND_BITS[kind], r,
                       first.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                       end.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), seed, rep0, n_reps, _dp(mean), _dp(m2))
    return mean.reshape(n_reps, M), m2.reshape(n_reps, M)


def mc_shared(N, S0, K, u, d, probs, kind, r, R, masses, seed, rep0=0, n_reps=1):
    probs = _probs(N, probs)
    masses = np.ascontiguousarray(masses, dtype=np.float64)
    M = 1 << r
    im = np.zeros(n_reps)
    isse = np.zeros(n_reps)
    sm = np.zeros(n_reps * M)
    lib().orc_mc_shared(N, S0, K, u, d, _dp(probs), KIND_BITS[kind], r, R, _dp(masses), seed, rep0, n_reps,
                        _dp(im), _dp(isse), _dp(sm))
    return im, isse, sm.reshape(n_reps, M)
