"""Exact expected value over all 2^N paths -- the drop-in engine entry points.

Reference: pkg/src/binpaths/exact.py.  Same names, signatures, return types
and exceptions as ``value_exact_serial`` (:103-109) and
``value_exact_parallel`` (:112-133); the validation order follows
``ValuationRequest.__post_init__`` (:48-56) and ``_check_enumerable``
(:75-80), so the same exception fires at the same point.

The 2^N sum runs in the CUDA engine (csrc/, via the C ABI in
include/binpaths_b200.h).  ``req.workers`` keeps its meaning as the
reference's rank count for validation, but the GPU result does not depend on
it: the engine reduces a fixed set of canonical super-blocks in a fixed
order, so ``value_exact_parallel(M=1) == value_exact_serial`` bit for bit for
every M (the reference guarantees this for M = 1 only, exact.py:116-118).
GPUs used: ``req.devices`` if the request carries it, else the
``BINPATHS_DEVICES`` environment variable (comma list), else device 0.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native
from .errors import (EnumerationGuard, InvalidInput, InvalidWorkerCount, LengthMismatch, NonConstantProbs,
                     PathDependentPayoff)
from .model import MarketInputs, TreeParams, leaf_prices
from .payoffs import BIT_TAG, PayoffLike, is_path_dependent, kind_bit, terminal_payoff

LARGE_DEPTH = 28      # exact.py:32 -- above this, enumeration needs force_large
CHUNK = 1 << 15       # exact.py:35 (reference batch size; kept for API parity)


def _positive_int(x) -> bool:
    return isinstance(x, int) and not isinstance(x, bool) and x >= 1


@dataclass(frozen=True)
class ValuationRequest:
    """One valuation: inputs, tree, payoff, worker count, guard override."""

    inputs: MarketInputs
    params: TreeParams
    kind: PayoffLike
    workers: int = 1
    force_large: bool = False

    def __post_init__(self):
        if not _positive_int(self.workers):
            raise InvalidWorkerCount(f"workers must be a positive integer, got {self.workers!r}")
        if self.params.n_steps != self.inputs.N:
            raise LengthMismatch(f"tree has {self.params.n_steps} steps but inputs say N={self.inputs.N}")


@dataclass
class ExactResult:
    """Full engine output for one valuation (beyond the reference's float)."""

    values: dict
    leaves: int
    code_sum: int
    hist: Optional[np.ndarray]
    kernel_ms: float
    engine: str
    inner_bits: int
    n_superblocks: int
    n_devices: int
    extra: dict = field(default_factory=dict)


def _check_enumerable(req) -> None:
    N = req.inputs.N
    if N > LARGE_DEPTH and not req.force_large:
        raise EnumerationGuard(
            f"N={N} means 2^{N} paths; pass the force-large override to enumerate beyond N={LARGE_DEPTH}")


def _devices(req) -> list:
    devs = getattr(req, "devices", None)
    if devs is None:
        env = os.environ.get("BINPATHS_DEVICES", "").strip()
        devs = [int(x) for x in env.split(",") if x.strip()] if env else [0]
    return [int(d) for d in devs]


def tree_of(req):
    """(BpTree, keep-alive) for a request; reads only the fields the reference
    engine reads: inputs.{S0,K,q,T,N}, params.{u,d,up_probs} (exact.py:87-99)."""
    inp, par = req.inputs, req.params
    N = int(inp.N)
    probs = np.asarray(par.up_probs, dtype=np.float64)
    if probs.shape != (N,):
        raise LengthMismatch(f"tree has {probs.shape[0]} steps but inputs say N={N}")
    S0 = float(inp.S0)
    if not math.isfinite(S0):  # any sign: the reference engine reads S0 unchecked (exact.py:96,99)
        raise InvalidInput(f"S0 must be a finite number, got {S0}")
    disc = math.exp(-float(inp.q) * float(inp.T))
    return _native.make_tree(N, S0, float(inp.K), float(par.u), float(par.d), disc, probs)


ENGINES = {0: "path-walk", 1: "affine-threshold", 2: "threshold-search", 3: "affine-threshold-weighted"}
_DEV_ARRAYS: dict = {}  # device tuple -> ctypes int array (read-only once built)
_MASK_BITS: dict = {}   # payoff mask -> its bits in ascending order


def value_exact(req, kinds: Optional[Sequence] = None, devices: Optional[Sequence[int]] = None,
                count: bool = False, generic: bool = False, search: bool = False) -> ExactResult:
    """Exact values of one or more payoff kinds in ONE pass over the 2^N paths.

    ``kinds`` defaults to ``[req.kind]``; ``count=True`` also returns the
    leaf bookkeeping (paths per up count, code checksum).  ``search=True``
    selects the threshold-search engine (K8): same exact value, but a node's
    inner leaves are counted by binary search instead of being visited, so
    its rate is an EFFECTIVE paths/s (not comparable to leaf evaluation).
    """
    _check_enumerable(req)
    kinds = [req.kind] if kinds is None else list(kinds)
    mask = 0
    for k in kinds:
        mask |= 1 << kind_bit(k)
    tree, keep = tree_of(req)
    devs = tuple(devices) if devices is not None else tuple(_devices(req))
    arr = _DEV_ARRAYS.get(devs)
    if arr is None:
        arr = _DEV_ARRAYS.setdefault(devs, (ctypes.c_int * len(devs))(*devs))
    res = _native.BpExactResult()
    flags = ((_native.FLAG_COUNT if count else 0) | (_native.FLAG_GENERIC if generic else 0)
             | (_native.FLAG_THRESHOLD if search else 0))
    L = _native.lib()
    _native.check(L.bp_exact(ctypes.byref(tree), mask, flags, len(devs), arr, ctypes.byref(res)))
    del keep
    bits = _MASK_BITS.get(mask)
    if bits is None:
        bits = _MASK_BITS.setdefault(mask, tuple(b for b in range(_native.N_PAYOFFS) if (mask >> b) & 1))
    vals = {BIT_TAG[b]: res.value[b] for b in bits}
    hist = np.array(res.hist[: req.inputs.N + 1], dtype=np.uint64) if count else None
    return ExactResult(values=vals, leaves=int(res.leaves), code_sum=int(res.code_sum), hist=hist,
                       kernel_ms=float(res.kernel_ms), engine=ENGINES[int(res.engine)],
                       inner_bits=int(res.inner_bits), n_superblocks=int(res.n_superblocks),
                       n_devices=int(res.n_devices))


def _single(req) -> float:
    res = value_exact(req)
    (value,) = res.values.values()
    return value


def value_exact_serial(req) -> float:
    """Full enumeration (exact.py:103-109); ignores req.workers."""
    return _single(req)


def value_exact_parallel(req) -> float:
    """Partitioned enumeration (exact.py:112-133) -- on the GPU(s)."""
    if not _positive_int(req.workers):
        raise InvalidWorkerCount(f"workers must be a positive integer, got {req.workers!r}")
    _check_enumerable(req)
    n = int(req.inputs.N)
    if req.workers > (1 << n):  # make_partition's bound (paths.py:117-120), checked before any launch
        raise InvalidWorkerCount(f"worker count {req.workers} exceeds the {1 << n} paths of an {n}-step tree")
    return _single(req)


def value_leaf_formula(req) -> float:
    """Closed form over the N+1 leaves for European kinds (exact.py:136-157).

    O(N) host arithmetic (not an enumeration): w_j = C(N,j) p^j (1-p)^(N-j)
    in log space.
    """
    if is_path_dependent(req.kind):
        raise PathDependentPayoff(
            f"{req.kind} depends on the whole path; the leaf formula only covers terminal-price payoffs")
    p = req.params.constant_up_prob()
    if p is None:
        raise NonConstantProbs("leaf formula needs one constant up probability across steps")
    n = req.inputs.N
    j = np.arange(n + 1)
    if p in (0.0, 1.0):
        weights = (j == (n if p == 1.0 else 0)).astype(np.float64)
    else:
        logc = np.array([math.lgamma(n + 1) - math.lgamma(k + 1) - math.lgamma(n - k + 1) for k in j])
        weights = np.exp(logc + j * math.log(p) + (n - j) * math.log1p(-p))
    values = terminal_payoff(req.kind, leaf_prices(req.params, req.inputs.S0), req.inputs.K)
    return math.exp(-req.inputs.q * req.inputs.T) * float(np.dot(weights, values))


_BP_TREE_DTYPE = np.dtype([(name, {ctypes.c_int32: "<i4", ctypes.c_double: "<f8", ctypes.c_void_p: "<u8"}[ct])
                           for name, ct in _native.BpTree._fields_], align=True)
assert _BP_TREE_DTYPE.itemsize == ctypes.sizeof(_native.BpTree)


def price_batch(N: int, S0, K, u, d, p, disc, kind, device: int = 0, with_time: bool = False):
    """Exact values of many independent trees (arrays, same N), one kind,
    one launch (bp_exact_batch).  Returns a numpy array (and kernel ms)."""
    arrs = np.broadcast_arrays(*(np.asarray(x, dtype=np.float64) for x in (S0, K, u, d, p, disc)))
    n = arrs[0].size
    S0a, Ka, ua, da, pa, da_ = (np.ascontiguousarray(a.reshape(-1)) for a in arrs)
    probs = np.ascontiguousarray(np.repeat(pa[:, None], N, axis=1))
    # the bp_tree array, filled column by column through a structured view of the same layout
    rec = np.zeros(n, dtype=_BP_TREE_DTYPE)
    rec["n_steps"] = int(N)
    for name, col in (("S0", S0a), ("K", Ka), ("u", ua), ("d", da), ("disc", da_)):
        rec[name] = col
    rec["up_probs"] = probs.ctypes.data + np.arange(n, dtype=np.uint64) * np.uint64(8 * int(N))
    trees = ctypes.cast(rec.ctypes.data, ctypes.POINTER(_native.BpTree))
    out = np.zeros(n)
    ms = ctypes.c_double()
    _native.check(_native.lib().bp_exact_batch(trees, n, 1 << kind_bit(kind), int(device), _native.dptr(out),
                                               ctypes.byref(ms)))
    return (out, ms.value) if with_time else out


def value_exact_batch(reqs: Sequence, kind=None, device: Optional[int] = None) -> np.ndarray:
    """value_exact_parallel over a list of requests (same N, constant p) in
    one launch.  Returns the values in request order."""
    reqs = list(reqs)
    if not reqs:
        return np.zeros(0)
    kind = reqs[0].kind if kind is None else kind
    N = int(reqs[0].inputs.N)
    for r in reqs:
        _check_enumerable(r)
        if int(r.inputs.N) != N:
            raise LengthMismatch("all requests of a batch must share N")
        if r.params.constant_up_prob() is None:
            raise NonConstantProbs("batched pricing needs one constant up probability per tree")
    cols = [(float(r.inputs.S0), float(r.inputs.K), float(r.params.u), float(r.params.d),
             float(r.params.up_probs[0]), math.exp(-float(r.inputs.q) * float(r.inputs.T))) for r in reqs]
    S0, K, u, d, p, disc = (np.array(c) for c in zip(*cols))
    dev = _devices(reqs[0])[0] if device is None else device
    return price_batch(N, S0, K, u, d, p, disc, kind, device=dev)
