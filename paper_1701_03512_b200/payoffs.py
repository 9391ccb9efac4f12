"""Payoff kinds and the callable plugin point (host side).

Reference: pkg/src/binpaths/payoffs.py.  ``PayoffKind`` keeps the reference's
four closed tags (:24-28).  The two BASELINE payoffs the reference reaches
only through its callable extension point (:33-34, 66-70) are exported as
callable objects with exactly that signature, ``(params, S0, K, path) ->
float``, so the REFERENCE engine can evaluate them too; each carries a
``kernel_bit`` the GPU engine dispatches on:

* ``ASIAN_CALL``         max(mean(S_1..S_N) - K, 0)
* ``FLOATING_LOOKBACK``  max(S_1..S_N) - S_N

Any other callable raises ``InvalidInput`` in the engines: there is no CPU
fallback.  ``payoff``/``payoff_batch`` evaluate single paths on the host
(reference API surface); the engines never call them.
"""
from __future__ import annotations

import enum
from typing import TYPE_CHECKING, Callable, Union

import numpy as np

from .errors import InvalidInput
from .model import asset_path

if TYPE_CHECKING:
    from .model import TreeParams
    from .paths import BernoulliPath


class PayoffKind(enum.Enum):
    EUROPEAN_CALL = "euro-call"
    EUROPEAN_PUT = "euro-put"
    ASIAN_PUT = "asian-put"
    FIXED_LOOKBACK_PUT = "lookback-put"


PAYOFF_NAMES = tuple(k.value for k in PayoffKind)
PayoffLike = Union[PayoffKind, Callable]

# tag -> bit position in the C ABI mask (include/binpaths_b200.h bp_payoff)
KIND_BIT = {
    "euro-call": 0,
    "euro-put": 1,
    "asian-put": 2,
    "lookback-put": 3,
    "asian-call": 4,
    "float-lookback": 5,
}
BIT_TAG = {v: k for k, v in KIND_BIT.items()}


class GpuPayoff:
    """A path functional the CUDA kernels implement, usable as a reference
    callable payoff (payoffs.py:66-70 signature)."""

    __slots__ = ("tag", "kernel_bit", "_fn")

    def __init__(self, tag: str, fn: Callable[[np.ndarray, float], float]):
        self.tag = tag
        self.kernel_bit = KIND_BIT[tag]
        self._fn = fn

    def __call__(self, params, S0, K, path) -> float:
        bits = np.asarray(path.bits(), dtype=bool)
        prices = S0 * np.cumprod(np.where(bits, params.u, params.d))
        return float(self._fn(prices, K))

    def __repr__(self) -> str:
        return f"GpuPayoff({self.tag!r})"

    def __reduce__(self):
        return (_gpu_payoff_by_tag, (self.tag,))


ASIAN_CALL = GpuPayoff("asian-call", lambda s, K: max(s.mean() - K, 0.0))
FLOATING_LOOKBACK = GpuPayoff("float-lookback", lambda s, K: s.max() - s[-1])
_BY_TAG = {p.tag: p for p in (ASIAN_CALL, FLOATING_LOOKBACK)}


def _gpu_payoff_by_tag(tag):
    return _BY_TAG[tag]


def parse_payoff(name: str) -> PayoffKind:
    """CLI tag -> kind; the tag set is closed exactly as in the reference (:39-46)."""
    for kind in PayoffKind:
        if kind.value == name:
            return kind
    raise InvalidInput(f"unknown payoff {name!r}; expected one of {', '.join(PAYOFF_NAMES)}")


def resolve_kind(name: str):
    """Extended lookup: the four tags plus 'asian-call' / 'float-lookback'."""
    if name in _BY_TAG:
        return _BY_TAG[name]
    return parse_payoff(name)


def kind_bit(kind) -> int:
    """Bit position of a kind in the C ABI mask.

    Accepts this package's kinds, the reference's ``PayoffKind`` members
    (matched by tag value, so a reference ``ValuationRequest`` drives the GPU
    engine unchanged) and ``GpuPayoff`` callables.  Anything else is an
    ``InvalidInput`` -- an arbitrary Python callable cannot run on the GPU.
    """
    bit = getattr(kind, "kernel_bit", None)
    if bit is not None:
        return int(bit)
    tag = getattr(kind, "value", None)
    if isinstance(tag, str) and tag in KIND_BIT and not callable(kind):
        return KIND_BIT[tag]
    raise InvalidInput(
        f"payoff {kind!r} has no GPU kernel; use a PayoffKind, ASIAN_CALL or FLOATING_LOOKBACK")


def is_path_dependent(kind: PayoffLike) -> bool:
    return kind_bit(kind) not in (0, 1) if _known(kind) else True


def _known(kind) -> bool:
    try:
        kind_bit(kind)
        return True
    except InvalidInput:
        return False


def terminal_payoff(kind: PayoffKind, terminal_prices: np.ndarray, K: float) -> np.ndarray:
    s = np.asarray(terminal_prices, dtype=np.float64)
    bit = kind_bit(kind)
    if bit == 0:
        return np.maximum(s - K, 0.0)
    if bit == 1:
        return np.maximum(K - s, 0.0)
    raise InvalidInput(f"{kind} is not a terminal-price payoff")


def _row_values(bit: int, prices: np.ndarray, K: float) -> np.ndarray:
    last = prices[..., -1]
    table = {
        0: lambda: np.maximum(last - K, 0.0),
        1: lambda: np.maximum(K - last, 0.0),
        2: lambda: np.maximum(K - prices.mean(axis=-1), 0.0),
        3: lambda: np.maximum(K - prices.min(axis=-1), 0.0),
        4: lambda: np.maximum(prices.mean(axis=-1) - K, 0.0),
        5: lambda: prices.max(axis=-1) - last,
    }
    return table[bit]()


def payoff(kind: PayoffLike, params: "TreeParams", S0: float, K: float, path: "BernoulliPath") -> float:
    """One payoff on one path (host helper, payoffs.py:66-80)."""
    if not _known(kind):
        return float(kind(params, S0, K, path))
    return float(_row_values(kind_bit(kind), asset_path(params, S0, path), K))


def payoff_batch(kind: PayoffLike, params: "TreeParams", S0: float, K: float, bits: np.ndarray) -> np.ndarray:
    """One payoff on a (batch, N) bit matrix (host helper, payoffs.py:83-113)."""
    bits = np.asarray(bits, dtype=bool)
    if bits.ndim != 2:
        raise InvalidInput(f"bit matrix must be 2-D, got shape {bits.shape}")
    if not _known(kind):
        from .paths import BernoulliPath
        return np.array([kind(params, S0, K, BernoulliPath.from_bits([int(b) for b in row])) for row in bits])
    prices = S0 * np.cumprod(np.where(bits, params.u, params.d), axis=1)
    return _row_values(kind_bit(kind), prices, K)
