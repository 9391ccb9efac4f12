"""The one-process-per-GPU path on a real device with a real NCCL process
group (world size 1 on the single GPU a gpurun box has): the ShardedExact
enqueue, the NCCL all_gather of the partials and the fixed-order combine,
against the single-call C-ABI valuation -- the plumbing bench.py uses under
torchrun for N > 1 (the multi-rank host logic is covered with gloo on CPU,
tests/test_dist_cpu.py)."""
import os
import socket

import pytest

import paper_1701_03512_b200 as bp
from paper_1701_03512_b200 import dist as bpd

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    yield dist
    dist.destroy_process_group()


def _req(N=24):
    P = bp.classic_crr(N, 0.2, 0.05, 1.0)
    inp = bp.MarketInputs(S0=100.0, K=105.0, q=0.05, sigma=0.2, T=1.0, N=N)
    return bp.ValuationRequest(inputs=inp, params=P, kind=bp.ASIAN_CALL, force_large=True)


def test_nccl_all_gather_and_combine_match_single_call(nccl_group):
    import torch
    from paper_1701_03512_b200.exact import tree_of
    req = _req()
    kinds = [bp.ASIAN_CALL, bp.FLOATING_LOOKBACK]
    want = bp.value_exact(req, kinds=kinds, devices=[0]).values
    tree, keep = tree_of(req)
    sh = bpd.ShardedExact(tree, keep, (1 << 4) | (1 << 5), 0, 1, 0)
    sh.enqueue()
    gathered = bpd.gather_partials(sh.local, sh.n_sb, 1)  # the NCCL collective itself
    torch.cuda.synchronize()
    got = bpd.combine(bpd.unpad(gathered.cpu().numpy(), sh.n_sb, 1), (1 << 4) | (1 << 5))
    assert got == want  # bitwise: same canonical super-blocks, same fixed-order combine
    sh.close()


def test_value_exact_distributed_world1(nccl_group):
    req = _req(26)
    want = bp.value_exact(req, devices=[0]).values
    # repeated calls reuse the cached sharded plan (first launches, then its graph): all bitwise equal
    for _ in range(3):
        assert bpd.value_exact_distributed(req, [bp.ASIAN_CALL], rank=0, world=1, device=0) == want
    other = _req(27)  # a different tree gets its own plan
    assert bpd.value_exact_distributed(other, [bp.ASIAN_CALL], rank=0, world=1, device=0) == \
        bp.value_exact(other, devices=[0]).values


def test_plan_enqueue_graph_replay_is_bitwise():
    """The first enqueue of a plan runs the launches, the second captures
    them as a graph, later ones replay it: all bitwise equal."""
    import torch
    from paper_1701_03512_b200.exact import tree_of
    req = _req(28)
    tree, keep = tree_of(req)
    mask = (1 << 4) | (1 << 5)
    sh = bpd.ShardedExact(tree, keep, mask, 0, 1, 0)
    outs = []
    for _ in range(4):
        sh.local.zero_()
        sh.enqueue()
        torch.cuda.synchronize()
        outs.append(bpd.combine(sh.local.cpu().numpy(), mask))
    assert outs[0] == outs[1] == outs[2] == outs[3]
    assert outs[0] == bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK], devices=[0]).values
    sh.close()
