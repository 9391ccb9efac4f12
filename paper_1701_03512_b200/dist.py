"""One process per GPU: shard the canonical super-blocks over ranks.

The exact sum over 2^N paths splits into at most 64 canonical super-blocks
(the top 6 bits of the unit index, csrc/bp_exact.cuh).  Rank g of G owns a
contiguous super-block range -- the paper's SPMD rank-prefix partition
(paths.py:103-123 with r = log2 G).  Each rank enqueues its
share on its own GPU (bp_exact_superblocks), the partials are exchanged with
ONE collective -- all_gather of a few hundred bytes over NCCL, the only
cross-GPU step (the paper's MPI.Reduce) -- and every rank
combines all partials in ascending super-block order, so the result is
bitwise identical for every G.

torch.distributed is plumbing here (process group, device buffers, NCCL);
the work is in the engine's kernels.  The combine logic is exercised on CPU
with the gloo backend (tests/test_dist_cpu.py).
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np

from . import _native
from .payoffs import BIT_TAG, kind_bit

N_PAYOFFS = _native.N_PAYOFFS


def shard_range(n_sb: int, rank: int, world: int) -> tuple:
    """Contiguous super-block range [first, first + count) of one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside [0, {world})")
    if world > n_sb:
        raise ValueError(f"{world} ranks exceed the {n_sb} super-blocks")
    base, extra = divmod(n_sb, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def shard_rows(n_sb: int, world: int) -> int:
    """Rows of every rank's exchange buffer: the largest shard, so the
    all_gather has equal counts for any world size (64 super-blocks over 3
    ranks: 22 / 21 / 21 real rows, all padded to 22)."""
    return -(-n_sb // world)


def combine(partials: np.ndarray, mask: int) -> dict:
    """Fixed-order (ascending super-block) compensated sum -> {tag: value},
    in the engine's host combine (bp_combine_superblocks); raises DeviceError
    when the engine library is missing (no Python fallback)."""
    p = np.ascontiguousarray(partials, dtype=np.float64).reshape(-1, N_PAYOFFS, 2)
    vals = np.zeros(N_PAYOFFS)
    _native.check(_native.lib().bp_combine_superblocks(_native.dptr(p), p.shape[0], mask, _native.dptr(vals)))
    return {BIT_TAG[k]: float(vals[k]) for k in range(N_PAYOFFS) if (mask >> k) & 1}


def gather_partials(local, n_sb: int, world: int, group=None):
    """all_gather of every rank's padded [shard_rows, 6, 2] partials (equal
    counts for any world size) -> [world * shard_rows, 6, 2]; unpad() keeps
    the real rows."""
    import torch
    import torch.distributed as dist

    per = local.shape[0]
    if per != shard_rows(n_sb, world):
        raise ValueError(f"exchange buffer has {per} rows, expected {shard_rows(n_sb, world)}")
    out = torch.empty((world * per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    return out


def unpad(gathered, n_sb: int, world: int):
    """The real rows of a gathered exchange buffer in rank order = ascending
    super-block order (rank g's rows are super-blocks shard_range(n_sb, g));
    numpy arrays and tensors alike."""
    per = shard_rows(n_sb, world)
    idx = np.concatenate([np.arange(g * per, g * per + shard_range(n_sb, g, world)[1]) for g in range(world)])
    return gathered[idx]


class ShardedExact:
    """Per-rank handle for repeated valuations of one tree (bench / serving).

    ``enqueue()`` launches this rank's super-blocks on the current torch CUDA
    stream; ``exchange()`` runs the NCCL all_gather; ``values()`` combines.
    """

    def __init__(self, tree, keep, mask: int, rank: int, world: int, device: int, flags: int = 0):
        import torch

        self.tree, self._keep, self.mask, self.flags = tree, keep, mask, flags
        self.rank, self.world, self.device = rank, world, device
        # prepared plan: tables built once, scratch reused across steps
        self._plan = ctypes.c_void_p()
        _native.check(_native.lib().bp_exact_plan_create(ctypes.byref(tree), mask, flags, ctypes.byref(self._plan)))
        n_sb, eng, L = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _native.check(_native.lib().bp_exact_plan_layout(self._plan, ctypes.byref(n_sb), ctypes.byref(eng),
                                                         ctypes.byref(L)))
        self.n_sb, self.engine, self.inner_bits = n_sb.value, eng.value, L.value
        self.first, self.count = shard_range(self.n_sb, rank, world)
        # padded to the largest shard: equal all_gather counts for any world size
        self.local = torch.zeros((shard_rows(self.n_sb, world), N_PAYOFFS, 2), dtype=torch.float64,
                                 device=f"cuda:{device}")
        self.gathered = None

    def enqueue(self, stream=None):
        import torch

        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        _native.check(_native.lib().bp_exact_plan_enqueue(
            self._plan, self.device, self.first, self.count, ctypes.c_void_p(self.local.data_ptr()), None,
            ctypes.c_void_p(st.cuda_stream)))

    def close(self):
        if self._plan:
            import torch
            torch.cuda.synchronize(self.device)
            _native.lib().bp_exact_plan_destroy(self._plan)
            self._plan = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def exchange(self, group=None):
        self.gathered = (gather_partials(self.local, self.n_sb, self.world, group) if self.world > 1
                         else self.local[:self.count])
        return self.gathered

    def values(self) -> dict:
        if self.gathered is None or self.world == 1:
            return combine(self.local[:self.count].detach().cpu().numpy(), self.mask)
        return combine(unpad(self.gathered.detach().cpu().numpy(), self.n_sb, self.world), self.mask)


_SHARDED_LRU: "collections.OrderedDict" = None
_SHARDED_CAP = 8


def _sharded_for(tree, keep, mask: int, rank: int, world: int, device: int, group) -> ShardedExact:
    """A cached ShardedExact per (contract, lattice, kinds, rank layout): a
    repeated valuation reuses its prepared plan -- and, from the second call
    on, the plan's captured CUDA graph."""
    import collections

    global _SHARDED_LRU
    if _SHARDED_LRU is None:
        _SHARDED_LRU = collections.OrderedDict()
    key = (bytes(tree)[:48], np.asarray(keep).tobytes(), mask, rank, world, device, id(group))
    sh = _SHARDED_LRU.get(key)
    if sh is not None:
        _SHARDED_LRU.move_to_end(key)
        return sh
    sh = ShardedExact(tree, keep, mask, rank, world, device)
    _SHARDED_LRU[key] = sh
    if len(_SHARDED_LRU) > _SHARDED_CAP:
        _, old = _SHARDED_LRU.popitem(last=False)
        old.close()
    return sh


def value_exact_distributed(req, kinds: Optional[Sequence] = None, rank: int = 0, world: int = 1,
                            device: int = 0, group=None) -> dict:
    """Exact values with this process as rank ``rank`` of ``world`` (one GPU each)."""
    from .exact import _check_enumerable, tree_of

    _check_enumerable(req)
    kinds = [req.kind] if kinds is None else list(kinds)
    mask = 0
    for k in kinds:
        mask |= 1 << kind_bit(k)
    tree, keep = tree_of(req)
    sh = _sharded_for(tree, keep, mask, rank, world, device, group)
    sh.enqueue()
    sh.exchange(group)
    return sh.values()


# ---------------------------------------------------------------------------
# Monte Carlo and batched pricing, one process per GPU.
#
# * Stratified MC with M >= G strata: rank g owns the contiguous strata range
#   of shard_range(M, g, G) -- the top log2 G bits of the k-bit prefix -- and
#   runs exactly the single-GPU work for them (same draws, same work items,
#   same per-stratum merge), so after the all_gather every stratum's
#   (theta_m, SSE_m) is bitwise the single-GPU value; the host combine
#   (mc._partitioned_from, ascending m) is unchanged.
# * M < G (basic MC, M = 1): every stratum's draws are split into G
#   contiguous, chunk-aligned ranges (bp_mc_range); the ranks' (n, mean, M2)
#   are merged with Chan's formula in rank order.  Equal to the single-GPU
#   statistics up to the association of that merge (~1e-15 relative).
# * Batched exact pricing: contiguous option slices, one all_gather.

def _gather_np(arr: np.ndarray, world: int, group=None) -> np.ndarray:
    """all_gather of an equal-shape float64 array -> [world, *shape] (NCCL on
    the current CUDA device, or gloo on CPU for the host-logic tests)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    local = torch.from_numpy(arr.reshape(-1)).to(dev)
    out = torch.empty(world * local.numel(), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(out, local, group=group)  # concatenated along dim 0
    return out.cpu().numpy().reshape((world,) + arr.shape)


def chunk_ranges(R: int, world: int, chunk: int) -> list:
    """[first, end) draw ranges of the G ranks: contiguous, starting at
    multiples of the engine's work-item size (so each rank's items are the
    single-GPU items), as balanced as the chunking allows."""
    n_chunks = -(-R // chunk) if R else 0
    out = []
    for g in range(world):
        c0, cn = (shard_range(n_chunks, g, world) if n_chunks >= world
                  else ((g, 1) if g < n_chunks else (n_chunks, 0)))
        out.append((min(c0 * chunk, R), min((c0 + cn) * chunk, R)))
    return out


def chan_merge(parts) -> tuple:
    """Fixed-order (rank order) Chan merge of (n, mean, M2) triples."""
    n, mean, m2 = 0.0, 0.0, 0.0
    for nb, mb, m2b in parts:
        if nb == 0:
            continue
        if n == 0:
            n, mean, m2 = float(nb), float(mb), float(m2b)
            continue
        tot = n + nb
        delta = mb - mean
        f = nb / tot
        mean = mean + delta * f
        m2 = m2 + m2b + delta * delta * n * f
        n = tot
    return n, mean, m2


def make_sharded_stats(rank: int, world: int, device: Optional[int] = None, group=None, compute=None):
    """A drop-in for mc._strata_stats that shards the work over `world`
    processes.  compute(req, r, first, end, seed, rep0, n_reps) -> (mean, m2)
    arrays [n_reps, 2^r] over draw ranges defaults to the GPU (bp_mc_range);
    the CPU host-logic tests pass the oracle."""
    from . import mc as _mc

    def native_compute(req, r, first, end, seed, rep0, n_reps):
        tree, keep = _mc._tree(req)
        M = 1 << r
        f = np.ascontiguousarray(first, dtype=np.uint64)
        e = np.ascontiguousarray(end, dtype=np.uint64)
        mean, m2 = np.zeros(n_reps * M), np.zeros(n_reps * M)
        ms = ctypes.c_double()
        dev = _mc._device(req) if device is None else device
        _native.check(_native.lib().bp_mc_range(ctypes.byref(tree), 1 << kind_bit(req.kind), r, _native.u64ptr(f),
                                                _native.u64ptr(e), seed, rep0, n_reps, dev, _native.dptr(mean),
                                                _native.dptr(m2), ctypes.byref(ms)))
        del keep
        return mean.reshape(n_reps, M), m2.reshape(n_reps, M)

    run = compute or native_compute

    def stats(req, r, draws, seed, rep0, n_reps):
        M = 1 << r
        draws = np.asarray(draws, dtype=np.uint64)
        if M >= world:  # strata shard: bitwise the single-GPU per-stratum statistics
            s0, cnt = shard_range(M, rank, world)
            end = np.zeros(M, dtype=np.uint64)
            end[s0:s0 + cnt] = draws[s0:s0 + cnt]
            mean, m2 = run(req, r, np.zeros(M, dtype=np.uint64), end, seed, rep0, n_reps)
            both = _gather_np(np.stack([mean, m2]), world, group) if world > 1 else np.stack([mean, m2])[None]
            theta, sse = np.zeros((n_reps, M)), np.zeros((n_reps, M))
            for g in range(world):
                a, c = shard_range(M, g, world)
                theta[:, a:a + c] = both[g, 0][:, a:a + c]
                sse[:, a:a + c] = both[g, 1][:, a:a + c]
            return theta, sse, 0.0
        # draw shard: every stratum's draws split by rank, Chan merge in rank order
        chunk = _native_chunk()
        rng = [chunk_ranges(int(R), world, chunk) for R in draws]
        first = np.array([rng[m][rank][0] for m in range(M)], dtype=np.uint64)
        end = np.array([rng[m][rank][1] for m in range(M)], dtype=np.uint64)
        mean, m2 = run(req, r, first, end, seed, rep0, n_reps)
        local = np.stack([mean, m2])
        both = _gather_np(local, world, group) if world > 1 else local[None]
        theta, sse = np.zeros((n_reps, M)), np.zeros((n_reps, M))
        for k in range(n_reps):
            for m in range(M):
                parts = [(rng[m][g][1] - rng[m][g][0], both[g, 0][k, m], both[g, 1][k, m]) for g in range(world)]
                _, theta[k, m], sse[k, m] = chan_merge(parts)
        return theta, sse, 0.0

    return stats


def _native_chunk() -> int:
    return 4096  # csrc/bp_mc_kernels.cu kChunk (work-item size in draws)


def run_repetitions_distributed(estimator, req, cfg, rank: int, world: int, device: Optional[int] = None,
                                group=None, compute=None):
    """mc.run_repetitions with the draws sharded over `world` processes (one
    GPU each); every rank returns the same RepetitionSummary.  Supports
    estimate_basic, estimate_partitioned and estimate_partitioned_equal (the
    shared-sample estimator evaluates one suffix sample under all strata and
    is not sharded here)."""
    from . import mc as _mc

    table = {_mc.estimate_basic: _mc._basic_reps, _mc.estimate_partitioned: _mc._partitioned_reps,
             _mc.estimate_partitioned_equal: _mc._equal_reps}
    if estimator not in table:
        from .errors import InvalidInput
        raise InvalidInput(f"{getattr(estimator, '__name__', estimator)} is not sharded across processes")
    stats = make_sharded_stats(rank, world, device, group, compute)
    estimates = tuple(table[estimator](req, cfg, 0, cfg.reps, stats=stats))
    values = np.array([e.value for e in estimates])
    variances = np.array([e.variance for e in estimates])
    return _mc.RepetitionSummary(estimates=estimates, mean_value=float(values.mean()),
                                 mean_variance=float(variances.mean()),
                                 empirical_variance=float(np.var(values, ddof=1)) if len(estimates) > 1 else 0.0)


def price_batch_distributed(N: int, S0, K, u, d, p, disc, kind, rank: int, world: int, device: int = 0, group=None,
                            compute=None) -> np.ndarray:
    """exact.price_batch with the options split into contiguous slices, one
    per process (GPU), and ONE all_gather of the per-option values.  Every
    rank returns all values in input order (each option's value is the same
    kernel work as in the single-GPU batch)."""
    from .exact import price_batch

    arrs = np.broadcast_arrays(*(np.asarray(x, dtype=np.float64) for x in (S0, K, u, d, p, disc)))
    n = arrs[0].size
    flat = [a.reshape(-1) for a in arrs]
    per = -(-n // world)
    lo, hi = min(rank * per, n), min((rank + 1) * per, n)
    run = compute or (lambda *a: price_batch(N, *a, kind, device=device))
    mine = np.zeros(per)
    if hi > lo:
        mine[:hi - lo] = run(*(x[lo:hi] for x in flat))
    allv = _gather_np(mine, world, group) if world > 1 else mine[None]
    return allv.reshape(-1)[:n]
