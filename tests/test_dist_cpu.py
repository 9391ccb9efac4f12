"""Multi-rank host logic with the gloo backend, world_size 2 (CPU only).

The GPU path (dist.ShardedExact) enqueues each rank's super-blocks and
exchanges the [count, 6, 2] partials with one all_gather; here the partials
come from the CPU oracle over the same code ranges, so the sharding, the
collective and the fixed-order combine are exercised without a GPU.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1701_03512_b200 import dist as bpd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_cover_superblocks():
    for n_sb in (1, 2, 8):
        for world in (1, 2, 4, 8):
            if world > n_sb:
                with pytest.raises(ValueError):
                    bpd.shard_range(n_sb, 0, world)
                continue
            seen = []
            for r in range(world):
                f, c = bpd.shard_range(n_sb, r, world)
                seen += list(range(f, f + c))
            assert seen == list(range(n_sb))


def _sb_partials(sbs, N=14):
    """Oracle partials of super-blocks `sbs` (top 3 code bits), kinds AC+FL."""
    import oracle
    u, p = 1.05, 0.52
    out = np.zeros((len(sbs), 6, 2))
    span = 1 << (N - 3)
    for i, sb in enumerate(sbs):
        v, _ = oracle.exact_range(N, 100.0, 101.0, u, 1 / u, p, math.exp(-0.05), ["asian-call", "float-lookback"],
                                  sb * span, (sb + 1) * span, 1)
        out[i, 4, 0] = v["asian-call"]
        out[i, 5, 0] = v["float-lookback"]
    return out


def _worker(rank, world, port, q):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = bpd.shard_range(8, rank, world)
    local = torch.from_numpy(_sb_partials(range(first, first + count)))
    gathered = bpd.gather_partials(local, world)
    vals = bpd.combine(gathered.numpy(), (1 << 4) | (1 << 5))
    q.put((rank, vals))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_exchange_is_bitwise_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=60) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    single = bpd.combine(_sb_partials(range(8)), (1 << 4) | (1 << 5))
    assert res[0] == res[1] == single
    import oracle
    full = oracle.exact(14, 100.0, 101.0, 1.05, 1 / 1.05, 0.52, math.exp(-0.05), ["asian-call", "float-lookback"])
    for k in full:
        assert single[k] == pytest.approx(full[k], rel=1e-13)
