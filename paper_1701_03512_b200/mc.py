"""Monte Carlo estimators -- drop-in for pkg/src/binpaths/mc.py.

Same names, signatures, return types and exceptions as the reference's
``estimate_basic`` (:135-159), ``estimate_partitioned`` (:234-257),
``estimate_partitioned_equal`` (:260-284), ``estimate_shared`` (:287-331),
``allocate_strata`` (:162-194) and ``run_repetitions`` (:334-353).

The draws and the per-stratum statistics (theta_m, SSE_m) run in the CUDA
engine (bp_mc_strata / bp_mc_shared).  The random stream is Philox4x32-10
keyed by (seed, stratum, rep) in its counter (include/binpaths_b200.h), the
GPU counterpart of the reference's mc_stream(seed, stratum, rep) keying:
reproducible, independent of thread / GPU mapping, M = 1 bit-identical to
basic MC.  Individual draws differ from numpy's Philox4x64 stream, so parity
with the reference is statistical (tests/test_mc_parity.py), while parity
with the CPU oracle, which draws the same bits, is to rounding.

Host-side arithmetic here is O(M): allocation, stratum masses and the
final combination, kept in the reference's order so per-stratum identities
(e.g. value == disc * sum(theta * mass)) hold bit for bit.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _native
from .errors import InfeasibleAllocation, InvalidInput, InvalidWorkerCount
from .paths import BernoulliPath, PathPartition, make_partition, partition_masses
from .payoffs import kind_bit


def _pos_int(x) -> bool:
    return isinstance(x, int) and not isinstance(x, bool)


@dataclass(frozen=True)
class McConfig:
    """Sampling plan: total draws R, stratum count M, seed, repetitions."""

    R: int
    M: int = 1
    seed: int = 0
    reps: int = 1

    def __post_init__(self):
        for name, lo in (("R", 1), ("M", 1), ("seed", 0), ("reps", 1)):
            v = getattr(self, name)
            if not _pos_int(v) or v < lo:
                want = "a nonnegative integer" if lo == 0 else "a positive integer"
                raise InvalidInput(f"{name} must be {want}, got {v!r}")


@dataclass(frozen=True)
class Estimate:
    value: float
    variance: float
    std_error: float
    R_used: int
    method: str
    seed: int
    per_stratum: Optional[tuple] = None


@dataclass(frozen=True)
class RepetitionSummary:
    estimates: tuple
    mean_value: float
    mean_variance: float
    empirical_variance: float

    @property
    def reps(self) -> int:
        return len(self.estimates)

    @property
    def values(self) -> np.ndarray:
        return np.array([e.value for e in self.estimates])

    @property
    def variances(self) -> np.ndarray:
        return np.array([e.variance for e in self.estimates])


# ---------------------------------------------------------------------------
class PhiloxStream:
    """Host view of the engine's stream (seed, stratum, rep): word q of draw
    i = Philox block q//4, lane q%4; bits() applies the engine's sampler.
    Mirrors mc_stream's role (mc.py:92-95) for inspection and tests; the
    estimators draw on the GPU."""

    def __init__(self, seed: int, stratum: int = 0, rep: int = 0):
        self.seed, self.stratum, self.rep = int(seed), int(stratum), int(rep)
        self._draw = 0

    def _block(self, j: int, c1: int) -> list:
        """Philox block with counter (j, c1, stratum, rep)."""
        key = (ctypes.c_uint32 * 2)(self.seed & 0xFFFFFFFF, self.seed >> 32)
        ctr = (ctypes.c_uint32 * 4)(j, c1, self.stratum, self.rep)
        blk = (ctypes.c_uint32 * 4)()
        _native.lib().bp_philox4x32_10(ctr, key, blk)
        return list(blk)

    def words(self, draw: int, count: int) -> np.ndarray:
        key = (ctypes.c_uint32 * 2)(self.seed & 0xFFFFFFFF, self.seed >> 32)
        out = np.empty(count, dtype=np.uint32)
        blk = (ctypes.c_uint32 * 4)()
        for j in range((count + 3) // 4):
            ctr = (ctypes.c_uint32 * 4)(j, draw, self.stratum, self.rep)
            _native.lib().bp_philox4x32_10(ctr, key, blk)
            n = min(4, count - 4 * j)
            out[4 * j:4 * j + n] = list(blk)[:n]
        return out

    LEVELS = 8  # threshold bits compared bit-sliced before the tie words (csrc/bp_mc_kernels.cu)

    def bits(self, probs: np.ndarray) -> np.ndarray:
        """Next draw's Bernoulli bits, bit t up with probability probs[t]
        (floor(p 2^32) / 2^32), by the engine's sampler with no fixed prefix:
        step w is bit w % 32 of group w // 32; the first of its 8 level bits
        (word 8 g + l) that is 1 decides it (up iff threshold bit 31 - l is
        1); with no 1 the group's next tie word does against the threshold's
        low 24 bits: the first tie of group g takes word 2 (i % 2) + g of the
        block (4, i // 2) that draws 2 j and 2 j + 1 share, the k-th (k >= 1)
        word 2 (k - 1) + g of the draw's own blocks 5, 6, ..."""
        probs = np.asarray(probs, dtype=np.float64)
        n = probs.shape[0]
        if n > 64:
            raise InvalidInput("the sampler draws at most 64 steps")
        L = self.LEVELS
        draw, self._draw = self._draw, self._draw + 1
        planes = [int(x) for x in self.words(draw, 2 * L)]
        up = np.zeros(n, dtype=bool)
        ties = [0, 0]
        for w in range(n):
            p = float(probs[w])
            if p >= 1.0:
                up[w] = True
                continue
            thr = int(math.floor(min(max(p, 0.0), 1.0) * 4294967296.0))
            g, b = divmod(w, 32)
            first = next((lvl for lvl in range(L) if (planes[L * g + lvl] >> b) & 1), None)
            if first is not None:
                up[w] = bool((thr >> (31 - first)) & 1)
                continue
            if ties[g] == 0:
                x = int(self._block(2 * L // 4, draw >> 1)[2 * (draw & 1) + g])
            else:
                q = 2 * (ties[g] - 1) + g
                x = int(self._block(2 * L // 4 + 1 + q // 4, draw)[q % 4])
            up[w] = x < ((thr << L) & 0xFFFFFFFF)
            ties[g] += 1
        return up

    def random(self, size: int) -> np.ndarray:
        """Uniforms of one draw's words (32-bit resolution)."""
        w = self.words(self._draw, int(size))
        self._draw += 1
        return w.astype(np.float64) / 4294967296.0


def mc_stream(seed: int, stratum: int = 0, rep: int = 0) -> PhiloxStream:
    return PhiloxStream(seed, stratum, rep)


def sample_path(params, rng: PhiloxStream) -> BernoulliPath:
    bits = rng.bits(params.up_probs)
    return BernoulliPath.from_bits([int(b) for b in bits])


# ---------------------------------------------------------------------------
def _discount(req) -> float:
    return math.exp(-req.inputs.q * req.inputs.T)


def _device(req) -> int:
    devs = getattr(req, "devices", None)
    if devs:
        return int(devs[0])
    import os
    env = os.environ.get("BINPATHS_DEVICES", "").strip()
    return int(env.split(",")[0]) if env else 0


def _tree(req):
    from .exact import tree_of
    return tree_of(req)


_PARTITIONS: dict = {}  # (n, M) -> the canonical prefix partition (immutable; a few entries)
_MASSES: dict = {}      # (n, M, prefix probabilities) -> stratum masses of that partition


def _stratified_partition(req, M: int) -> PathPartition:
    if M & (M - 1) != 0:
        raise InvalidWorkerCount(f"stratum count must be a power of two, got {M}")
    n = int(req.inputs.N)
    hit = _PARTITIONS.get((n, M))
    if hit is not None:
        return hit
    if n > 62:  # MC only: 63/64-step paths (BASELINE config 4), prefix strata as in make_partition
        r = M.bit_length() - 1
        if r > n:
            raise InvalidWorkerCount(f"stratum count {M} exceeds the paths of an {n}-step tree")
        part = PathPartition(n=n, m=M, prefix_width=r, blocks=tuple((i,) for i in range(M)))
    else:
        part = make_partition(n, M)
    if len(_PARTITIONS) >= 8:
        _PARTITIONS.clear()
    _PARTITIONS[(n, M)] = part
    return part


def _stratum_masses(req, part: PathPartition) -> list:
    """partition_masses of a _stratified_partition, remembered per lattice
    prefix (repeated estimates on one tree: 4096 strata cost ~2 ms in Python)."""
    probs = np.asarray(req.params.up_probs, dtype=np.float64)
    key = (part.n, part.m, probs[:part.prefix_width].tobytes(), probs.shape[0])
    hit = _MASSES.get(key)
    if hit is None:
        hit = partition_masses(req.params, part)
        if len(_MASSES) >= 8:
            _MASSES.clear()
        _MASSES[key] = hit
    return hit


def _strata_stats(req, r: int, draws, seed: int, rep0: int, n_reps: int):
    """(theta[n_reps, M], sse[n_reps, M], kernel_ms) from the GPU."""
    tree, keep = _tree(req)
    M = 1 << r
    d = np.ascontiguousarray(draws, dtype=np.uint64)
    theta = np.zeros(n_reps * M)
    sse = np.zeros(n_reps * M)
    ms = ctypes.c_double()
    _native.check(_native.lib().bp_mc_strata(ctypes.byref(tree), 1 << kind_bit(req.kind), r, _native.u64ptr(d),
                                             seed, rep0, n_reps, _device(req), _native.dptr(theta),
                                             _native.dptr(sse), ctypes.byref(ms)))
    del keep
    return theta.reshape(n_reps, M), sse.reshape(n_reps, M), ms.value


def allocate_strata(partition: PathPartition, params, R: int) -> list:
    """Largest-remainder split of R draws proportional to stratum mass,
    >= 1 draw for every positive-mass stratum, ties to the lower rank
    (mc.py:162-194)."""
    masses = partition_masses(params, partition)
    positive = [m for m in range(partition.m) if masses[m] > 0.0]
    if R < len(positive):
        raise InfeasibleAllocation(f"R={R} draws cannot cover {len(positive)} strata with positive mass")
    targets = R * np.asarray(masses, dtype=np.float64)  # the same IEEE products as R * w per stratum
    base = np.floor(targets)
    # largest remainders first, ties to the lower stratum: primary key floor - target, then m
    order = np.lexsort((np.arange(partition.m), base - targets))
    alloc = [int(x) for x in base]
    for m in order[: R - sum(alloc)].tolist():
        alloc[m] += 1
    floor_of = [1 if w > 0.0 else 0 for w in masses]
    while True:
        starved = next((m for m in positive if alloc[m] == 0), None)
        if starved is None:
            return alloc
        donor = max(range(partition.m), key=lambda m: (alloc[m] - floor_of[m], -m))
        alloc[donor] -= 1
        alloc[starved] += 1


def _basic_from(req, cfg, theta, sse) -> Estimate:
    disc = _discount(req)
    variance = disc * disc * (sse / (cfg.R * cfg.R))
    return Estimate(value=disc * theta, variance=variance, std_error=math.sqrt(variance), R_used=cfg.R,
                    method="basic", seed=cfg.seed)


def _partitioned_from(req, cfg, masses, alloc, thetas, sses, equal: bool) -> Estimate:
    disc = _discount(req)
    w = np.asarray(masses, dtype=np.float64)
    th = np.asarray(thetas, dtype=np.float64)
    if equal:
        var_theta = float(np.sum(w * w * np.asarray(sses) / (cfg.R * cfg.R)))
    else:
        var_theta = float(np.sum(np.asarray(sses))) / (cfg.R * cfg.R)
    variance = disc * disc * var_theta
    return Estimate(value=disc * float(np.sum(th * w)), variance=variance, std_error=math.sqrt(variance),
                    R_used=int(sum(alloc)), method="partitioned", seed=cfg.seed,
                    per_stratum=tuple(zip(range(len(alloc)), map(int, alloc), th.tolist())))


def _basic_reps(req, cfg, rep0, n_reps, stats=None):
    if cfg.R < 2:
        raise InvalidInput(f"basic estimator needs R >= 2, got {cfg.R}")
    theta, sse, _ = (stats or _strata_stats)(req, 0, [cfg.R], cfg.seed, rep0, n_reps)
    return [_basic_from(req, cfg, float(theta[k, 0]), float(sse[k, 0])) for k in range(n_reps)]


def _partitioned_reps(req, cfg, rep0, n_reps, stats=None):
    if cfg.R < cfg.M:
        raise InfeasibleAllocation(f"partitioned estimator needs R >= M, got R={cfg.R}, M={cfg.M}")
    part = _stratified_partition(req, cfg.M)
    masses = _stratum_masses(req, part)
    alloc = allocate_strata(part, req.params, cfg.R)
    theta, sse, _ = (stats or _strata_stats)(req, part.prefix_width, alloc, cfg.seed, rep0, n_reps)
    return [_partitioned_from(req, cfg, masses, alloc, theta[k], sse[k], equal=False) for k in range(n_reps)]


def _equal_reps(req, cfg, rep0, n_reps, stats=None):
    part = _stratified_partition(req, cfg.M)
    masses = _stratum_masses(req, part)
    alloc = [cfg.R] * cfg.M
    theta, sse, _ = (stats or _strata_stats)(req, part.prefix_width, alloc, cfg.seed, rep0, n_reps)
    return [_partitioned_from(req, cfg, masses, alloc, theta[k], sse[k], equal=True) for k in range(n_reps)]


def _shared_reps(req, cfg, rep0, n_reps):
    if cfg.R < 2:
        raise InvalidInput(f"shared estimator needs R >= 2, got {cfg.R}")
    part = _stratified_partition(req, cfg.M)
    masses = np.array(_stratum_masses(req, part))
    tree, keep = _tree(req)
    im = np.zeros(n_reps)
    isse = np.zeros(n_reps)
    sm = np.zeros(n_reps * cfg.M)
    ms = ctypes.c_double()
    _native.check(_native.lib().bp_mc_shared(ctypes.byref(tree), 1 << kind_bit(req.kind), part.prefix_width, cfg.R,
                                             _native.dptr(masses), cfg.seed, rep0, n_reps, _device(req),
                                             _native.dptr(im), _native.dptr(isse), _native.dptr(sm),
                                             ctypes.byref(ms)))
    del keep
    sm = sm.reshape(n_reps, cfg.M)
    disc = _discount(req)
    out = []
    for k in range(n_reps):
        variance = disc * disc * (float(isse[k]) / (cfg.R * cfg.R))
        out.append(Estimate(value=disc * float(im[k]), variance=variance, std_error=math.sqrt(variance),
                            R_used=cfg.R, method="shared", seed=cfg.seed,
                            per_stratum=tuple(zip(range(cfg.M), [cfg.R] * cfg.M, sm[k].tolist()))))
    return out


def estimate_basic(req, cfg: McConfig, rep: int = 0) -> Estimate:
    """Plain MC: R i.i.d. paths on stream (seed, 0, rep) (mc.py:135-159)."""
    return _basic_reps(req, cfg, rep, 1)[0]


def estimate_partitioned(req, cfg: McConfig, rep: int = 0, eval_threads: int = 1) -> Estimate:
    """Stratified MC, proportional allocation (mc.py:234-257).  eval_threads
    is accepted for API parity; results never depend on it."""
    return _partitioned_reps(req, cfg, rep, 1)[0]


def estimate_partitioned_equal(req, cfg: McConfig, rep: int = 0, eval_threads: int = 1) -> Estimate:
    """Stratified MC, R draws in every stratum (mc.py:260-284)."""
    return _equal_reps(req, cfg, rep, 1)[0]


def estimate_shared(req, cfg: McConfig, rep: int = 0, eval_threads: int = 1) -> Estimate:
    """Shared-sample MC: one suffix sample under every prefix (mc.py:287-331)."""
    return _shared_reps(req, cfg, rep, 1)[0]


_BATCHED = {
    estimate_basic: _basic_reps,
    estimate_partitioned: _partitioned_reps,
    estimate_partitioned_equal: _equal_reps,
    estimate_shared: _shared_reps,
}


def run_repetitions(estimator: Callable, req, cfg: McConfig, **estimator_kwargs) -> RepetitionSummary:
    """cfg.reps repetitions keyed by rep = 0..reps-1 (mc.py:334-353).

    For this package's estimators all repetitions run in ONE launch (the rep
    index is part of the Philox counter); the estimates are bit-identical to
    calling the estimator once per rep.
    """
    batched = _BATCHED.get(estimator)
    if batched is not None:
        estimates = tuple(batched(req, cfg, 0, cfg.reps))
    else:
        estimates = tuple(estimator(req, cfg, rep=k, **estimator_kwargs) for k in range(cfg.reps))
    values = np.array([e.value for e in estimates])
    variances = np.array([e.variance for e in estimates])
    return RepetitionSummary(estimates=estimates, mean_value=float(values.mean()),
                             mean_variance=float(variances.mean()),
                             empirical_variance=float(np.var(values, ddof=1)) if len(estimates) > 1 else 0.0)
