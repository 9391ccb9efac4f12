"""Multi-rank host logic with the gloo backend, world sizes 2 and 3 (CPU only).

The GPU path (dist.ShardedExact) enqueues each rank's super-blocks and
exchanges its padded [shard_rows, 6, 2] partials with one all_gather; here the
partials come from the CPU oracle over the same code ranges, so the sharding
(including world sizes that do not divide the 64 super-blocks), the
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

N_SB = 64
N = 14


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_cover_superblocks():
    for n_sb in (1, 2, 8, 64):
        for world in (1, 2, 3, 4, 5, 7, 8):
            if world > n_sb:
                with pytest.raises(ValueError):
                    bpd.shard_range(n_sb, 0, world)
                continue
            seen = []
            for r in range(world):
                f, c = bpd.shard_range(n_sb, r, world)
                assert c <= bpd.shard_rows(n_sb, world)
                seen += list(range(f, f + c))
            assert seen == list(range(n_sb))


def test_unpad_keeps_real_rows_in_superblock_order():
    for world in (1, 2, 3, 5, 7):
        per = bpd.shard_rows(N_SB, world)
        padded = np.full((world * per, 6, 2), -1.0)
        for g in range(world):
            f, c = bpd.shard_range(N_SB, g, world)
            padded[g * per:g * per + c, 0, 0] = np.arange(f, f + c)
        got = bpd.unpad(padded, N_SB, world)
        assert got.shape == (N_SB, 6, 2)
        assert list(got[:, 0, 0]) == list(range(N_SB))


def _sb_partials(sbs):
    """Oracle partials of super-blocks `sbs` (top 6 code bits), kinds AC+FL."""
    import oracle
    u, p = 1.05, 0.52
    out = np.zeros((len(sbs), 6, 2))
    span = 1 << (N - 6)
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
    first, count = bpd.shard_range(N_SB, rank, world)
    local = torch.zeros((bpd.shard_rows(N_SB, world), 6, 2), dtype=torch.float64)
    local[:count] = torch.from_numpy(_sb_partials(range(first, first + count)))
    gathered = bpd.gather_partials(local, N_SB, world)
    vals = bpd.combine(bpd.unpad(gathered.numpy(), N_SB, world), (1 << 4) | (1 << 5))
    q.put((rank, vals))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchange_is_bitwise_single_rank(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=90) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    single = bpd.combine(_sb_partials(range(N_SB)), (1 << 4) | (1 << 5))
    assert all(res[r] == single for r in range(world))
    import oracle
    full = oracle.exact(N, 100.0, 101.0, 1.05, 1 / 1.05, 0.52, math.exp(-0.05), ["asian-call", "float-lookback"])
    for k in full:
        assert single[k] == pytest.approx(full[k], rel=1e-13)


def test_gather_rejects_unpadded_buffer():
    import torch
    with pytest.raises(ValueError):
        bpd.gather_partials(torch.zeros((21, 6, 2), dtype=torch.float64), N_SB, 3)
