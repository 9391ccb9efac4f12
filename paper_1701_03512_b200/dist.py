"""One process per GPU: shard the canonical super-blocks over ranks.

The exact sum over 2^N paths splits into at most 8 canonical super-blocks
(the top 3 bits of the node index, csrc/bp_exact.cuh).  Rank g of G owns a
contiguous super-block range -- the paper's SPMD rank-prefix partition
(paths.py:103-123 with r = log2 G).  Each rank enqueues its
share on its own GPU (bp_exact_superblocks), the partials are exchanged with
ONE collective -- all_gather of a few hundred bytes over NCCL, the only
cross-GPU step (the paper's MPI.Reduce) -- and every rank
combines all partials in ascending super-block order, so the result is
bitwise identical for G = 1, 2, 4, 8.

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


def combine(partials: np.ndarray, mask: int) -> dict:
    """Fixed-order (ascending super-block) compensated sum -> {tag: value}."""
    p = np.ascontiguousarray(partials, dtype=np.float64).reshape(-1, N_PAYOFFS, 2)
    vals = np.zeros(N_PAYOFFS)
    if _native.available():
        _native.check(_native.lib().bp_combine_superblocks(_native.dptr(p), p.shape[0], mask, _native.dptr(vals)))
    else:  # the same TwoSum merge in Python (host logic tests without the .so)
        for k in range(N_PAYOFFS):
            if not (mask >> k) & 1:
                continue
            s = c = 0.0
            for b in range(p.shape[0]):
                s2, c2 = float(p[b, k, 0]), float(p[b, k, 1])
                t = s + s2
                bp = t - s
                e = (s - (t - bp)) + (s2 - bp)
                s, c = t, c + (c2 + e)
            vals[k] = s + c
    return {BIT_TAG[k]: float(vals[k]) for k in range(N_PAYOFFS) if (mask >> k) & 1}


def gather_partials(local, world: int, group=None):
    """all_gather of each rank's [count, 6, 2] partial tensor (equal counts)."""
    import torch
    import torch.distributed as dist

    out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    return out


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
        self.local = torch.zeros((self.count, N_PAYOFFS, 2), dtype=torch.float64, device=f"cuda:{device}")
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
        self.gathered = gather_partials(self.local, self.world, group) if self.world > 1 else self.local
        return self.gathered

    def values(self) -> dict:
        src = self.gathered if self.gathered is not None else self.local
        return combine(src.detach().cpu().numpy(), self.mask)


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
    sh = ShardedExact(tree, keep, mask, rank, world, device)
    sh.enqueue()
    sh.exchange(group)
    return sh.values()
