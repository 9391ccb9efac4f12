"""Per-rank parity and reference-route parity of the exact engine (GPU).

* rank g of G (G = 2^r) owns the codes
  [g 2^{N-r}, (g+1) 2^{N-r}) (paths.py:141-145); its partial must equal the
  reference's _rank_value(req, make_partition(N, G), g) (exact.py:83-100) --
  here the oracle's discounted sum over the same code range -- to 1e-12.
* Duck-typed inputs with S0 <= 0 (the reference reads inputs.S0 unchecked,
  exact.py:96,99): the sign-flip oracle routes of SURVEY §8(c) run through
  the drop-in and match the reference's own route values in the goldens.
* count=True with per-step probabilities (leaf bookkeeping on the path walk).
"""
import math
from types import SimpleNamespace

import numpy as np
import pytest

import oracle
import paper_1701_03512_b200 as bp
from conftest import load_golden
from paper_1701_03512_b200 import dist as bpd
from paper_1701_03512_b200.exact import tree_of

pytestmark = pytest.mark.gpu

REL = 1e-12
K2 = 105.47846749285817  # config 2's strike (default_rng(0).uniform(80, 120))
KINDS = ["asian-call", "float-lookback"]


def _req(N, K=K2):
    P = bp.classic_crr(N, 0.2, 0.05, 1.0)
    inp = bp.MarketInputs(S0=100.0, K=K, q=0.05, sigma=0.2, T=1.0, N=N)
    return bp.ValuationRequest(inputs=inp, params=P, kind=bp.ASIAN_CALL, force_large=True), P


@pytest.mark.parametrize("N", [24, 30])
def test_rank_partials_match_oracle_ranges(N):
    import torch
    req, P = _req(N)
    tree, keep = tree_of(req)
    mask = (1 << 4) | (1 << 5)
    # the oracle over the 8 finest rank ranges (coarser ranks are unions)
    span = 1 << (N - 3)
    fine = [oracle.exact_range(N, 100.0, K2, P.u, P.d, P.up_probs[0], math.exp(-0.05), KINDS, g * span,
                               (g + 1) * span, 16)[0] for g in range(8)]
    for G in (2, 4, 8):
        per = 8 // G
        for g in range(G):
            sh = bpd.ShardedExact(tree, keep, mask, g, G, 0)
            sh.enqueue()
            torch.cuda.synchronize()
            got = sh.values()  # this rank's super-blocks only (no exchange)
            sh.close()
            lo_sb, cnt = bpd.shard_range(sh.n_sb, g, G)
            assert lo_sb * (1 << N) // sh.n_sb == g * (1 << N) // G  # same code range as make_partition
            for k in KINDS:
                want = sum(fine[i][k] for i in range(g * per, (g + 1) * per))
                assert abs(got[k] - want) <= REL * abs(want), (N, G, g, k, got[k], want)


def test_sign_flip_routes_through_the_drop_in():
    """Asian call = ASIAN_PUT at (-S0, -K); floating lookback =
    FIXED_LOOKBACK_PUT(-S0, 0) - EUROPEAN_CALL(S0, 0): the reference's own
    values of these routes are in tests/golden/exact_small.json."""
    g = load_golden("exact_small.json")
    n = 0
    for case in g["cases"]:
        if "route_asian_call" not in case:
            continue
        N = case["N"]
        probs = np.asarray(case.get("up_probs", [case.get("p")] * N), dtype=np.float64)
        P = bp.TreeParams(dt=case["T"] / N, u=case["u"], d=case["d"], beta=0.5 * (case["u"] + case["d"]),
                          up_probs=probs)

        def value(kind, S0, K):
            inputs = SimpleNamespace(S0=S0, K=K, q=case["q"], T=case["T"], N=N)
            return bp.value_exact_parallel(bp.ValuationRequest(inputs=inputs, params=P, kind=kind, workers=2,
                                                               force_large=True))

        ac = value(bp.PayoffKind.ASIAN_PUT, -case["S0"], -case["K"])
        fl = value(bp.PayoffKind.FIXED_LOOKBACK_PUT, -case["S0"], 0.0) - \
            value(bp.PayoffKind.EUROPEAN_CALL, case["S0"], 0.0)
        for got, want in ((ac, case["route_asian_call"]), (fl, case["route_float_lookback"])):
            assert abs(got - want) <= max(REL * abs(want), 1e-13), (case["tag"], got, want)
        n += 1
    assert n > 10


def test_nonpositive_spot_takes_the_path_walk():
    _, P = _req(18)
    inputs = SimpleNamespace(S0=-100.0, K=-90.0, q=0.05, T=1.0, N=18)
    r = bp.value_exact(bp.ValuationRequest(inputs=inputs, params=P, kind=bp.PayoffKind.ASIAN_PUT,
                                           force_large=True))
    assert r.engine == "path-walk"
    want = oracle.exact(18, -100.0, -90.0, P.u, P.d, P.up_probs[0], math.exp(-0.05), ["asian-put"])
    assert abs(r.values["asian-put"] - want["asian-put"]) <= REL * abs(want["asian-put"])


def test_count_with_custom_probs_uses_the_path_walk():
    N = 18
    rng = np.random.default_rng(5)
    probs = rng.uniform(0.3, 0.7, N)
    u = 1.05
    P = bp.TreeParams(dt=1.0 / N, u=u, d=1 / u, beta=0.5 * (u + 1 / u), up_probs=probs)
    inp = bp.MarketInputs(S0=100.0, K=101.0, q=0.05, sigma=0.2, T=1.0, N=N)
    req = bp.ValuationRequest(inputs=inp, params=P, kind=bp.ASIAN_CALL, force_large=True)
    r = bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK], count=True)
    assert r.engine == "path-walk"
    assert [int(x) for x in r.hist] == [math.comb(N, h) for h in range(N + 1)]
    assert r.leaves == 1 << N
    want = oracle.exact(N, 100.0, 101.0, u, 1 / u, probs, math.exp(-0.05), KINDS)
    fast = bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK])  # the weighted class engine
    for k in KINDS:
        assert abs(r.values[k] - want[k]) <= REL * abs(want[k])
        assert abs(fast.values[k] - want[k]) <= REL * abs(want[k])
