"""Sharded Monte Carlo and batched pricing across processes,
host logic with the gloo backend at world size 2 and 3 on CPU.  The
per-rank compute is the CPU oracle over the same draw ranges the GPU ranks
would run (bp_mc_range), so the strata split, the chunk-aligned draw split,
the all_gather and the rank-order Chan merge are exercised without a GPU.

* strata shard (M >= G): every stratum's statistics bitwise equal the
  single-process run;
* draw shard (basic MC): equal up to the Chan-merge association (1e-12);
* batched pricing: every option's value bitwise the single-process value.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

N, S0, K, U, P = 12, 100.0, 100.0, 1.08, 0.52


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _req():
    import paper_1701_03512_b200 as bp
    params = bp.TreeParams(dt=1.0 / N, u=U, d=1 / U, beta=0.5 * (U + 1 / U), up_probs=np.full(N, P))
    inputs = bp.MarketInputs(S0=S0, K=K, q=0.03, sigma=0.2, T=1.0, N=N)
    return bp.ValuationRequest(inputs=inputs, params=params, kind=bp.ASIAN_CALL)


def _oracle_compute(req, r, first, end, seed, rep0, n_reps):
    import oracle
    return oracle.mc_range(N, S0, K, U, 1 / U, P, "asian-call", r, first, end, seed, rep0, n_reps)


def _oracle_batch(S0s, Ks, us, ds, ps, discs):
    import oracle
    return np.array([oracle.exact(N, s, k, u, d, p, disc, ["asian-call"])["asian-call"]
                     for s, k, u, d, p, disc in zip(S0s, Ks, us, ds, ps, discs)])


def _batch_inputs():
    rng = np.random.default_rng(5)
    n = 7
    return (rng.uniform(80, 120, n), rng.uniform(80, 120, n), np.full(n, U), np.full(n, 1 / U), np.full(n, P),
            np.full(n, math.exp(-0.03)))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1701_03512_b200 as bp
    from paper_1701_03512_b200 import dist as bpd
    req = _req()
    out = {}
    for name, est, cfg in (("equal", bp.estimate_partitioned_equal, bp.McConfig(R=300, M=4, seed=9, reps=3)),
                           ("prop", bp.estimate_partitioned, bp.McConfig(R=9000, M=8, seed=9, reps=2)),
                           ("basic", bp.estimate_basic, bp.McConfig(R=10000, seed=4, reps=2))):
        s = bpd.run_repetitions_distributed(est, req, cfg, rank, world, compute=_oracle_compute)
        out[name] = [(e.value, e.variance) for e in s.estimates]
    out["batch"] = bpd.price_batch_distributed(N, *_batch_inputs(), bp.ASIAN_CALL, rank, world,
                                               compute=_oracle_batch).tolist()
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_mc_and_batch_match_single_process(world):
    import paper_1701_03512_b200 as bp
    from paper_1701_03512_b200 import dist as bpd
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert all(res[r] == res[0] for r in range(world))  # every rank holds the same result
    got = res[0]
    # single process: the same estimators over full ranges (world 1, no collective)
    req = _req()

    def single(est, cfg):
        s = bpd.run_repetitions_distributed(est, req, cfg, 0, 1, compute=_oracle_compute)
        return [(e.value, e.variance) for e in s.estimates]

    assert got["equal"] == single(bp.estimate_partitioned_equal, bp.McConfig(R=300, M=4, seed=9, reps=3))
    if world <= 8:
        assert got["prop"] == single(bp.estimate_partitioned, bp.McConfig(R=9000, M=8, seed=9, reps=2))
    want = single(bp.estimate_basic, bp.McConfig(R=10000, seed=4, reps=2))
    for (v, var), (v1, var1) in zip(got["basic"], want):
        assert v == pytest.approx(v1, rel=1e-12) and var == pytest.approx(var1, rel=1e-12)
    assert got["batch"] == _oracle_batch(*_batch_inputs()).tolist()


def test_chunk_ranges_cover_and_align():
    from paper_1701_03512_b200 import dist as bpd
    for R in (0, 1, 4095, 4096, 10000, 1 << 20):
        for world in (1, 2, 3, 8):
            rs = bpd.chunk_ranges(R, world, 4096)
            assert rs[0][0] == 0 and rs[-1][1] == R
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(f % 4096 == 0 or f == R for f, _ in rs)


def test_chan_merge_matches_two_pass():
    from paper_1701_03512_b200 import dist as bpd
    rng = np.random.default_rng(0)
    x = rng.normal(3.0, 2.0, 1000)
    parts = []
    for a, b in ((0, 300), (300, 301), (301, 301), (301, 1000)):
        seg = x[a:b]
        parts.append((len(seg), seg.mean() if len(seg) else 0.0, ((seg - seg.mean()) ** 2).sum() if len(seg) else 0.0))
    n, mean, m2 = bpd.chan_merge(parts)
    assert n == 1000 and mean == pytest.approx(x.mean(), rel=1e-14)
    assert m2 == pytest.approx(((x - x.mean()) ** 2).sum(), rel=1e-12)
