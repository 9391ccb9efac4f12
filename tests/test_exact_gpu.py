"""GPU parity of the exact engine against the CPU oracle and the reference goldens.

Bar (BASELINE.json north_star): exact values within 1e-12 relative; leaf
bookkeeping (paths per up count, total, code checksum) bit-exact.
"""
import math
import os

import numpy as np
import pytest

import oracle
import paper_1701_03512_b200 as bp
from conftest import load_golden

pytestmark = pytest.mark.gpu

ALL = ["euro-call", "euro-put", "asian-put", "lookback-put", "asian-call", "float-lookback"]
REL = 1e-12


def _req(N, S0, K, q, T, u, d, probs, kind=bp.ASIAN_CALL, force=True):
    params = bp.TreeParams(dt=T / N, u=u, d=d, beta=0.5 * (u + d), up_probs=np.broadcast_to(probs, (N,)))
    inputs = bp.MarketInputs(S0=S0, K=K, q=q, sigma=0.2, T=T, N=N)
    return bp.ValuationRequest(inputs=inputs, params=params, kind=kind, force_large=force)


def _close(got, want, rel=REL, abs_=1e-13):
    return abs(got - want) <= max(rel * abs(want), abs_)


@pytest.mark.parametrize("generic", [False, True])
def test_small_cases_all_kinds_vs_goldens(generic):
    g = load_golden("exact_small.json")
    for case in g["cases"] + g["medium"]:
        N = case["N"]
        probs = case.get("up_probs", [case.get("p")] * N)
        req = _req(N, case["S0"], case["K"], case["q"], case["T"], case["u"], case["d"], np.array(probs))
        res = bp.value_exact(req, kinds=[bp.resolve_kind(k) for k in ALL], generic=generic)
        for k in ALL:
            want = case["values"][k]
            assert _close(res.values[k], want), (case["tag"], k, res.values[k], want)


def test_config1_goldens_and_bookkeeping():
    g = load_golden("exact_config1.json")
    req = _req(20, 100.0, 100.0, 0.05, 1.0, g["u"], g["d"], g["p"])
    res = bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK, bp.PayoffKind.ASIAN_PUT,
                                     bp.PayoffKind.FIXED_LOOKBACK_PUT], count=True)
    assert res.engine == "affine-threshold"
    assert _close(res.values["asian-call"], g["asian_call"])
    assert _close(res.values["float-lookback"], g["float_lookback"])
    assert _close(res.values["asian-put"], g["asian_put"])
    assert _close(res.values["lookback-put"], g["fixed_lookback_put"])
    assert [int(x) for x in res.hist] == [math.comb(20, h) for h in range(21)]
    assert res.leaves == 1 << 20
    assert res.code_sum == ((1 << 19) * ((1 << 20) - 1)) % (1 << 64)


@pytest.mark.parametrize("N", [16, 17, 20, 23, 24])
def test_fast_engine_matches_oracle(N):
    rng = np.random.default_rng(N)
    for _ in range(3):
        S0 = float(rng.uniform(50, 150)); K = float(S0 * rng.uniform(0.8, 1.2))
        r = float(rng.uniform(0.0, 0.08)); sigma = float(rng.uniform(0.1, 0.6)); T = float(rng.uniform(0.25, 3))
        P = bp.classic_crr(N, sigma, r, T)
        req = _req(N, S0, K, r, T, P.u, P.d, P.up_probs[0])
        res = bp.value_exact(req, kinds=[bp.resolve_kind(k) for k in ALL], count=True)
        want = oracle.exact(N, S0, K, P.u, P.d, P.up_probs[0], math.exp(-r * T), ALL, workers=16)
        for k in ALL:
            assert _close(res.values[k], want[k]), (N, k, res.values[k], want[k])
        assert [int(x) for x in res.hist] == [math.comb(N, h) for h in range(N + 1)]


def test_engines_agree_and_are_deterministic():
    P = bp.classic_crr(22, 0.3, 0.03, 2.0)
    req = _req(22, 100.0, 105.0, 0.03, 2.0, P.u, P.d, P.up_probs[0])
    kinds = [bp.resolve_kind(k) for k in ALL]
    a = bp.value_exact(req, kinds=kinds)
    b = bp.value_exact(req, kinds=kinds)
    c = bp.value_exact(req, kinds=kinds, generic=True)
    for k in ALL:
        assert a.values[k] == b.values[k]  # bitwise repeatable
        assert _close(a.values[k], c.values[k]), (k, a.values[k], c.values[k])


def test_drop_in_entry_points():
    g = load_golden("exact_config1.json")
    P = bp.classic_crr(20, 0.2, 0.05, 1.0)
    inputs = bp.MarketInputs(S0=100.0, K=100.0, q=0.05, sigma=0.2, T=1.0, N=20)
    for workers in (1, 2, 3, 8):
        req = bp.ValuationRequest(inputs=inputs, params=P, kind=bp.ASIAN_CALL, workers=workers)
        v = bp.value_exact_parallel(req)
        assert v == bp.value_exact_serial(req)
        assert _close(v, g["asian_call"])


def test_config2_golden_N30_two_payoffs_one_pass():
    g = load_golden("exact_config2.json")
    req = _req(30, 100.0, g["K"], 0.05, 1.0, g["u"], g["d"], g["p"])
    res = bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK])
    assert res.engine == "affine-threshold"
    assert _close(res.values["asian-call"], g["asian_call"]), (res.values, g["asian_call"])
    assert _close(res.values["float-lookback"], g["float_lookback"]), (res.values, g["float_lookback"])


@pytest.mark.parametrize("N", [20, 30])
def test_superblock_sharding_is_bitwise_invariant_across_G(N):
    """Emulate G = 1, 2, 4, 8 ranks on one GPU: every rank's super-block range
    is enqueued separately (bp_exact_superblocks) and the gathered partials
    are combined in fixed order -- identical bits for every G."""
    import torch
    from paper_1701_03512_b200 import dist as bpd
    from paper_1701_03512_b200.exact import tree_of
    P = bp.classic_crr(N, 0.2, 0.05, 1.0)
    req = _req(N, 100.0, 103.0, 0.05, 1.0, P.u, P.d, P.up_probs[0])
    tree, keep = tree_of(req)
    mask = (1 << 4) | (1 << 5)
    results = {}
    for G in (1, 2, 4, 8):
        parts = []
        for rank in range(G):
            sh = bpd.ShardedExact(tree, keep, mask, rank, G, 0)
            sh.enqueue()
            torch.cuda.synchronize()
            parts.append(sh.local.cpu().numpy())
        results[G] = bpd.combine(np.concatenate(parts), mask)
    assert results[1] == results[2] == results[4] == results[8]
    single = bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK])
    assert single.values == results[1]
    # the in-process multi-device path (one host thread per listed device)
    twin = bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK], devices=[0, 0, 0, 0])
    assert twin.values == results[1] and twin.n_devices == 4


def test_bookkeeping_code_checksum_large_N():
    P = bp.classic_crr(28, 0.2, 0.05, 1.0)
    req = _req(28, 100.0, 100.0, 0.05, 1.0, P.u, P.d, P.up_probs[0])
    res = bp.value_exact(req, kinds=[bp.ASIAN_CALL], count=True)
    N = 28
    assert res.leaves == 1 << N
    assert res.code_sum == ((1 << (N - 1)) * ((1 << N) - 1)) % (1 << 64)
    assert [int(x) for x in res.hist] == [math.comb(N, h) for h in range(N + 1)]


def test_guard_and_extreme_lattices():
    # guard fires before the launch
    P = bp.classic_crr(30, 0.2, 0.05, 1.0)
    with pytest.raises(bp.EnumerationGuard):
        bp.value_exact_serial(_req(30, 100.0, 100.0, 0.05, 1.0, P.u, P.d, P.up_probs[0], force=False))
    # heavy-tailed beta-CRR desk (sigma = 3): fast engine vs path walk
    inputs = bp.MarketInputs(S0=20.0, K=100.0, q=0.06, sigma=3.0, T=1.0, N=18)
    D = bp.derive_crr(inputs)
    req = bp.ValuationRequest(inputs=inputs, params=D, kind=bp.PayoffKind.ASIAN_PUT)
    kinds = [bp.resolve_kind(k) for k in ALL]
    a = bp.value_exact(req, kinds=kinds)
    b = bp.value_exact(req, kinds=kinds, generic=True)
    assert a.engine == "affine-threshold"
    for k in ALL:
        assert _close(a.values[k], b.values[k]), (k, a.values[k], b.values[k])


def test_paper_values_N32_beta_crr():
    """PAPER.md:389,534 exact values (82.115 / 93.196), reproduced by the
    reference's own enumeration (tests/golden/exact_paper.json) -- matched to 1e-12."""
    g = load_golden("exact_paper.json")
    inputs = bp.MarketInputs(S0=g["S0"], K=g["K"], q=g["q"], sigma=g["sigma"], T=g["T"], N=32)
    params = bp.derive_crr(inputs)
    assert params.u == g["u"] and params.up_probs[0] == g["p"]
    req = bp.ValuationRequest(inputs=inputs, params=params, kind=bp.PayoffKind.ASIAN_PUT, force_large=True)
    res = bp.value_exact(req, kinds=[bp.PayoffKind.ASIAN_PUT, bp.PayoffKind.FIXED_LOOKBACK_PUT])
    for tag in ("asian-put", "lookback-put"):
        assert _close(res.values[tag], g["values"][tag]), (tag, res.values[tag], g["values"][tag])
        assert round(res.values[tag], 3) == g["published"][tag]


def test_config3_golden_N36_when_available():
    import os
    from conftest import GOLDEN
    if not os.path.exists(os.path.join(GOLDEN, "exact_config3.json")):
        pytest.skip("config 3 golden not generated yet (tools/make_goldens.py config3, ~90 min)")
    g = load_golden("exact_config3.json")
    req = _req(36, 100.0, 105.0, 0.03, 2.0, g["u"], g["d"], g["p"])
    res = bp.value_exact(req, kinds=[bp.ASIAN_CALL])
    assert _close(res.values["asian-call"], g["asian_call"]), (res.values, g["asian_call"])


@pytest.mark.parametrize("N", [16, 20, 24, 30])
def test_threshold_search_engine_matches_leaf_engine(N):
    """K8 (binary search over class-sorted tables) gives the
    same exact value as the explicit leaf engine K1 and the oracle."""
    rng = np.random.default_rng(100 + N)
    S0 = float(rng.uniform(50, 150)); K = float(S0 * rng.uniform(0.85, 1.15))
    r = float(rng.uniform(0.0, 0.08)); sigma = float(rng.uniform(0.1, 0.5)); T = float(rng.uniform(0.25, 3))
    P = bp.classic_crr(N, sigma, r, T)
    req = _req(N, S0, K, r, T, P.u, P.d, P.up_probs[0])
    kinds = [bp.resolve_kind(k) for k in ALL]
    a = bp.value_exact(req, kinds=kinds)
    b = bp.value_exact(req, kinds=kinds, search=True)
    assert b.engine == "threshold-search"
    for k in ALL:
        assert _close(b.values[k], a.values[k]), (N, k, a.values[k], b.values[k])


def test_threshold_search_config_goldens():
    g1 = load_golden("exact_config2.json")
    req = _req(30, 100.0, g1["K"], 0.05, 1.0, g1["u"], g1["d"], g1["p"])
    res = bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK], search=True)
    assert _close(res.values["asian-call"], g1["asian_call"])
    assert _close(res.values["float-lookback"], g1["float_lookback"])
    g = load_golden("exact_paper.json")
    inputs = bp.MarketInputs(S0=g["S0"], K=g["K"], q=g["q"], sigma=g["sigma"], T=g["T"], N=32)
    req = bp.ValuationRequest(inputs=inputs, params=bp.derive_crr(inputs), kind=bp.PayoffKind.ASIAN_PUT,
                              force_large=True)
    res = bp.value_exact(req, kinds=[bp.PayoffKind.ASIAN_PUT, bp.PayoffKind.FIXED_LOOKBACK_PUT], search=True)
    for tag in ("asian-put", "lookback-put"):
        assert _close(res.values[tag], g["values"][tag]), (tag, res.values[tag], g["values"][tag])


@pytest.mark.parametrize("N", [16, 19, 22])
def test_per_step_probabilities_weighted_engine(N):
    """with_custom_probs trees (model.py:152-161): the per-leaf-weight engine K1w
    vs the oracle and the path-walk engine, every kind."""
    rng = np.random.default_rng(7 + N)
    inputs = bp.MarketInputs(S0=50.0, K=51.0, q=0.02, sigma=0.35, T=1.5, N=N)
    params = bp.with_custom_probs(inputs, rng.uniform(0.25, 0.75, size=N))
    req = bp.ValuationRequest(inputs=inputs, params=params, kind=bp.ASIAN_CALL, force_large=True)
    kinds = [bp.resolve_kind(k) for k in ALL]
    a = bp.value_exact(req, kinds=kinds)
    assert a.engine == "affine-threshold-weighted"
    b = bp.value_exact(req, kinds=kinds, generic=True)
    want = oracle.exact(N, 50.0, 51.0, params.u, params.d, params.up_probs, math.exp(-0.02 * 1.5), ALL, workers=8)
    for k in ALL:
        assert _close(a.values[k], want[k]), (N, k, a.values[k], want[k])
        assert _close(b.values[k], want[k]), (N, k, b.values[k], want[k])


@pytest.mark.parametrize("seed", range(6))
def test_fuzz_general_lattices_vs_oracle(seed):
    """Seeded fuzz over lattices the BASELINE configs do not reach: d != 1/u,
    p near 0 or 1, deep in/out of the money strikes; the leaf engine (K1),
    the threshold-search engine (K8) and the oracle must agree (1e-12)."""
    rng = np.random.default_rng(1000 + seed)
    N = int(rng.integers(16, 23))
    u = float(rng.uniform(1.005, 1.25))
    d = float(rng.uniform(0.75, 0.999)) if seed % 2 else 1.0 / u
    p = float(rng.choice([rng.uniform(0.01, 0.05), rng.uniform(0.2, 0.8), rng.uniform(0.95, 0.99)]))
    S0 = float(rng.uniform(10, 200))
    K = float(S0 * rng.choice([0.3, rng.uniform(0.9, 1.1), 2.5]))
    q, T = float(rng.uniform(-0.02, 0.1)), float(rng.uniform(0.1, 4.0))
    req = _req(N, S0, K, q, T, u, d, p)
    kinds = [bp.resolve_kind(k) for k in ALL]
    res = bp.value_exact(req, kinds=kinds, count=True)
    assert res.engine == "affine-threshold"
    want = oracle.exact(N, S0, K, u, d, p, math.exp(-q * T), ALL, workers=16)
    for k in ALL:
        assert _close(res.values[k], want[k]), (seed, N, k, res.values[k], want[k])
    assert [int(x) for x in res.hist] == [math.comb(N, h) for h in range(N + 1)]
    srch = bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK], search=True)
    for k in ("asian-call", "float-lookback"):
        assert _close(srch.values[k], want[k]), (seed, "search", k, srch.values[k], want[k])


def test_graph_replay_is_bitwise_the_launch_path():
    """Repeated synchronous valuations replay a captured CUDA graph (bp_capi.cu
    try_graph_job); the values must be bitwise those of the ordinary launch
    path (BINPATHS_GRAPH=0, a fresh process) and stable across replays and
    across contracts sharing the lattice."""
    import json
    import subprocess
    import sys
    from conftest import ROOT
    code = ("import json, paper_1701_03512_b200 as bp\n"
            "P = bp.classic_crr(26, 0.2, 0.05, 1.0)\n"
            "out = []\n"
            "for K in (95.0, 105.0, 95.0):\n"
            "    inp = bp.MarketInputs(S0=100.0, K=K, q=0.05, sigma=0.2, T=1.0, N=26)\n"
            "    req = bp.ValuationRequest(inputs=inp, params=P, kind=bp.ASIAN_CALL, force_large=True)\n"
            "    for _ in range(3):\n"
            "        out.append(bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK]).values)\n"
            "print(json.dumps([[v.hex() for v in d.values()] for d in out]))\n")
    runs = {}
    for flag in ("1", "0"):
        env = dict(os.environ, BINPATHS_GRAPH=flag)
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT,
                           timeout=300)
        assert p.returncode == 0, p.stderr
        runs[flag] = json.loads(p.stdout.strip().splitlines()[-1])
    assert runs["1"] == runs["0"]
    r = runs["1"]
    assert r[0] == r[1] == r[2] == r[6] == r[7] == r[8] and r[3] == r[4] == r[5] and r[0] != r[3]


@pytest.mark.parametrize("u", [1.0 + 1e-7, 1.0 + 1e-4, 1.6])
def test_screen_code_collisions_vs_oracle(u):
    """Stress of the I15 screen's exact fallback (bp_leaf.cuh I15Class): at
    u = 1 + 1e-7 every class's values fit in a few 15-bit codes, so nearly
    every threshold shares a code with many leaves and the boundary fix and
    the walk decide most leaves in fp64; at u = 1.6 the classes span a wide
    range.  Every kind, K around the money so thresholds fall inside the
    classes; K1 against the oracle and against the path walk (1e-12)."""
    N, S0 = 18, 100.0
    d = 1.0 / u
    for K in (99.99, 100.0, 100.02, 140.0):
        req = _req(N, S0, K, 0.01, 1.0, u, d, 0.5)
        kinds = [bp.resolve_kind(k) for k in ALL]
        res = bp.value_exact(req, kinds=kinds)
        assert res.engine == "affine-threshold"
        walk = bp.value_exact(req, kinds=kinds, generic=True)
        want = oracle.exact(N, S0, K, u, d, 0.5, math.exp(-0.01), ALL, workers=16)
        for k in ALL:
            assert _close(res.values[k], want[k]), (u, K, k, res.values[k], want[k])
            assert _close(res.values[k], walk.values[k]), (u, K, k, res.values[k], walk.values[k])
