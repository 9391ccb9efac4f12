"""GPU side of the sharded Monte Carlo: bp_mc_range over the
ranks' draw / strata ranges reproduces the single-GPU statistics -- strata
subsets bitwise, chunk-aligned draw splits after the rank-order Chan merge
to 1e-12 -- and matches the oracle draw for draw.  The multi-rank exchange
itself is covered with gloo on CPU (tests/test_dist_mc_cpu.py) and with a
real NCCL group of one rank here."""
import ctypes
import os
import socket

import numpy as np
import pytest

import oracle
import paper_1701_03512_b200 as bp
from paper_1701_03512_b200 import _native
from paper_1701_03512_b200 import dist as bpd
from paper_1701_03512_b200 import mc as bmc

pytestmark = pytest.mark.gpu


def _req(N=64, kind=None):
    P = bp.classic_crr(N, 0.2, 0.05, 1.0)
    from types import SimpleNamespace
    inputs = SimpleNamespace(S0=100.0, K=100.0, q=0.05, T=1.0, N=N)
    req = object.__new__(bp.ValuationRequest)
    for f, v in dict(inputs=inputs, params=P, kind=kind or bp.ASIAN_CALL, workers=1, force_large=True).items():
        object.__setattr__(req, f, v)
    return req


def _range(req, r, first, end, seed, rep0=0, n_reps=1):
    tree, keep = bmc._tree(req)
    M = 1 << r
    f = np.ascontiguousarray(first, dtype=np.uint64)
    e = np.ascontiguousarray(end, dtype=np.uint64)
    mean, m2 = np.zeros(n_reps * M), np.zeros(n_reps * M)
    _native.check(_native.lib().bp_mc_range(ctypes.byref(tree), 1 << 4, r, _native.u64ptr(f), _native.u64ptr(e),
                                            seed, rep0, n_reps, 0, _native.dptr(mean), _native.dptr(m2),
                                            ctypes.byref(ctypes.c_double())))
    return mean.reshape(n_reps, M), m2.reshape(n_reps, M)


def test_strata_subsets_are_bitwise_the_full_run():
    req, r, R = _req(), 6, 5000
    theta, sse, _ = bmc._strata_stats(req, r, [R] * 64, 11, 0, 2)
    for world in (2, 4, 8):
        for g in range(world):
            s0, cnt = bpd.shard_range(64, g, world)
            end = np.zeros(64, dtype=np.uint64)
            end[s0:s0 + cnt] = R
            mean, m2 = _range(req, r, np.zeros(64), end, 11, 0, 2)
            assert np.array_equal(mean[:, s0:s0 + cnt], theta[:, s0:s0 + cnt])
            assert np.array_equal(m2[:, s0:s0 + cnt], sse[:, s0:s0 + cnt])


@pytest.mark.parametrize("world", [2, 3, 8])
def test_basic_mc_draw_split_merges_to_the_full_run(world):
    req, R = _req(), 3 * 4096 * 5 + 123
    theta, sse, _ = bmc._strata_stats(req, 0, [R], 5, 0, 1)
    parts = []
    for f, e in bpd.chunk_ranges(R, world, 4096):
        mean, m2 = _range(req, 0, [f], [e], 5)
        parts.append((e - f, mean[0, 0], m2[0, 0]))
    n, mean, m2 = bpd.chan_merge(parts)
    assert n == R
    assert mean == pytest.approx(theta[0, 0], rel=1e-12) and m2 == pytest.approx(sse[0, 0], rel=1e-12)


def test_range_matches_oracle_draw_for_draw():
    req = _req(N=20)
    P = req.params
    first, end = [4096, 0, 8192, 100], [4096 + 777, 50, 8192 + 4096, 4196]
    mean, m2 = _range(req, 2, first, end, 3)
    om, o2 = oracle.mc_range(20, 100.0, 100.0, P.u, P.d, P.up_probs[0], "asian-call", 2, first, end, 3)
    assert np.allclose(mean, om, rtol=1e-12, atol=1e-14) and np.allclose(m2, o2, rtol=1e-11, atol=1e-12)


def test_unaligned_ranges_match_oracle_draw_for_draw():
    """Ranges starting or ending at odd draws: a draw's tie words come from the
    pair block it shares with its neighbour whether or not that neighbour is
    in the range (an odd start walks the range draw by draw)."""
    req = _req(N=40)
    P = req.params
    first, end = [4097, 1, 8191, 101], [4097 + 778, 50, 8191 + 4097, 4196]
    mean, m2 = _range(req, 2, first, end, 3)
    om, o2 = oracle.mc_range(40, 100.0, 100.0, P.u, P.d, P.up_probs[0], "asian-call", 2, first, end, 3)
    assert np.allclose(mean, om, rtol=1e-12, atol=1e-14) and np.allclose(m2, o2, rtol=1e-11, atol=1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_distributed_estimators_through_nccl_world1():
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        req = _req(N=32)
        cfg = bp.McConfig(R=512, M=4096, seed=2, reps=3)
        got = bpd.run_repetitions_distributed(bp.estimate_partitioned_equal, req, cfg, 0, 1, device=0)
        want = bp.run_repetitions(bp.estimate_partitioned_equal, req, cfg)
        assert [e.value for e in got.estimates] == [e.value for e in want.estimates]
        vals = bpd.price_batch_distributed(24, [100.0, 90.0], [100.0, 95.0], 1.02, 1 / 1.02, 0.51, 0.97,
                                           bp.ASIAN_CALL, 0, 1, device=0)
        assert vals.tolist() == bp.price_batch(24, [100.0, 90.0], [100.0, 95.0], 1.02, 1 / 1.02, 0.51, 0.97,
                                               bp.ASIAN_CALL).tolist()
    finally:
        dist.destroy_process_group()
