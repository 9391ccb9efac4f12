"""Host-side mirror of the reference API (CPU only, no GPU calls).

Pinned against the golden vectors made from the reference (partitions,
allocations, block masses, derive_crr) and the reference's own error
behaviour.  Engine calls that need a GPU are only checked for raising
before any launch (guard / validation order) or loudly without a device.
"""
import math
import os
import sys

import numpy as np
import pytest

import paper_1701_03512_b200 as bp
from conftest import load_golden


def test_derive_crr_matches_reference_bitwise():
    for c in load_golden("exact_small.json")["derive_crr"]:
        P = bp.derive_crr(bp.MarketInputs(S0=1.0, K=1.0, q=c["q"], sigma=c["sigma"], T=c["T"], N=c["N"]))
        assert (P.dt, P.u, P.d, P.beta, float(P.up_probs[0])) == (c["dt"], c["u"], c["d"], c["beta"], c["p"])


def test_frozen_crr_values():
    # reference tests/test_model.py:20-29
    P = bp.derive_crr(bp.MarketInputs(S0=5.0, K=10.0, q=0.06, sigma=0.30, T=1.0, N=2))
    assert P.beta == pytest.approx(1.02416484221657, rel=1e-13)
    assert P.u == pytest.approx(1.245329088948476, rel=1e-13)
    assert P.d == pytest.approx(0.8030005954846637, rel=1e-13)
    assert P.up_probs[0] == pytest.approx(0.5142195038978686, rel=1e-13)


def test_classic_crr_matches_baseline_lattice():
    g = load_golden("exact_config1.json")
    P = bp.classic_crr(20, 0.2, 0.05, 1.0)
    assert P.u == g["u"] and P.d == g["d"] and P.up_probs[0] == g["p"]


def test_partitions_match_reference():
    for c in load_golden("exact_small.json")["partitions"]:
        part = bp.make_partition(c["n"], c["m"])
        assert part.prefix_width == c["prefix_width"]
        assert [list(b) for b in part.blocks] == c["blocks"]
        covered = sorted(code for r in range(part.m) for lo, hi in bp.block_code_ranges(part, r)
                         for code in range(lo, hi)) if c["n"] <= 12 else None
        if covered is not None:
            assert covered == list(range(1 << c["n"]))


def test_allocations_and_masses_match_reference_bitwise():
    for c in load_golden("exact_small.json")["allocations"]:
        P = bp.TreeParams(dt=1.0, u=1.1, d=1 / 1.1, beta=1.0, up_probs=np.array(c["up_probs"]))
        part = bp.make_partition(c["n"], c["m"])
        assert bp.allocate_strata(part, P, c["R"]) == c["alloc"]
        assert [bp.block_probability(P, part, k) for k in range(c["m"])] == c["masses"]


def test_allocation_infeasible():
    P = bp.TreeParams(dt=1.0, u=2.0, d=0.5, beta=1.25, up_probs=np.full(6, 0.5))
    with pytest.raises(bp.InfeasibleAllocation):
        bp.allocate_strata(bp.make_partition(6, 4), P, 3)


def test_bit_order_and_round_trip():
    p = bp.BernoulliPath.from_bits([1, 0, 0, 1, 1])
    assert p.code == 0b10011 and p.bits() == (1, 0, 0, 1, 1)
    for code in range(1 << 7):
        assert bp.BernoulliPath.from_bits(bp.BernoulliPath(code, 7).bits()).code == code
    bits = bp.codes_to_bits(np.arange(8, dtype=np.uint64), 3)
    assert bits.tolist()[5] == [True, False, True]
    with pytest.raises(bp.InvalidInput):
        bp.BernoulliPath(code=8, n=3)


def test_market_input_domains():
    for bad in (dict(S0=0.0), dict(K=-1.0), dict(sigma=-0.1), dict(T=0.0), dict(N=0), dict(N=63), dict(q=math.inf)):
        kw = dict(S0=1.0, K=1.0, q=0.0, sigma=0.2, T=1.0, N=4)
        kw.update(bad)
        with pytest.raises(bp.InvalidInput):
            bp.MarketInputs(**kw)
    with pytest.raises(bp.LengthMismatch):
        bp.with_custom_probs(bp.MarketInputs(S0=1.0, K=1.0, q=0.0, sigma=0.2, T=1.0, N=3), [0.5, 0.5])
    with pytest.raises(bp.ProbabilityOutOfRange):
        bp.with_custom_probs(bp.MarketInputs(S0=1.0, K=1.0, q=0.0, sigma=0.2, T=1.0, N=2), [0.5, 1.0])


def _req(N=30, kind=bp.ASIAN_CALL, workers=1, force=False):
    inp = bp.MarketInputs(S0=100.0, K=100.0, q=0.05, sigma=0.2, T=1.0, N=N)
    return bp.ValuationRequest(inputs=inp, params=bp.classic_crr(N, 0.2, 0.05, 1.0), kind=kind, workers=workers,
                               force_large=force)


def test_guard_and_validation_fire_before_any_launch():
    with pytest.raises(bp.EnumerationGuard):
        bp.value_exact_serial(_req(29))
    with pytest.raises(bp.EnumerationGuard):
        bp.value_exact_parallel(_req(40, workers=8))
    with pytest.raises(bp.InvalidWorkerCount):
        _req(10, workers=0)
    with pytest.raises(bp.InvalidWorkerCount):  # make_partition's m <= 2^N bound (paths.py:115-118)
        bp.value_exact_parallel(_req(2, workers=5))
    with pytest.raises(bp.LengthMismatch):
        bp.ValuationRequest(inputs=bp.MarketInputs(S0=1.0, K=1.0, q=0.0, sigma=0.2, T=1.0, N=5),
                            params=bp.classic_crr(4, 0.2, 0.0, 1.0), kind=bp.ASIAN_CALL)


def test_unknown_callable_payoff_is_rejected_not_run_on_cpu():
    def my_payoff(params, S0, K, path):
        return 0.0
    with pytest.raises(bp.InvalidInput):
        bp.kind_bit(my_payoff)
    with pytest.raises(bp.InvalidInput):
        bp.value_exact_serial(_req(10, kind=my_payoff))


def test_engine_fails_loudly_without_gpu():
    from paper_1701_03512_b200 import _native
    if _native.available() and _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(bp.PricingError):
        bp.value_exact_serial(_req(10))


def test_parse_payoff_is_closed_like_the_reference():
    assert bp.parse_payoff("asian-put") is bp.PayoffKind.ASIAN_PUT
    with pytest.raises(bp.InvalidInput):
        bp.parse_payoff("asian-call")
    assert bp.resolve_kind("asian-call") is bp.ASIAN_CALL


def test_gpu_payoffs_are_reference_callables_and_match_goldens():
    """ASIAN_CALL / FLOATING_LOOKBACK have the reference callable signature;
    evaluated by the host helper they reproduce the reference's values."""
    g = load_golden("exact_small.json")
    case = next(c for c in g["cases"] if c["tag"] == "N5_classic")
    P = bp.TreeParams(dt=1.0, u=case["u"], d=case["d"], beta=1.0, up_probs=np.array(case["up_probs"]))
    for kind, tag in ((bp.ASIAN_CALL, "asian-call"), (bp.FLOATING_LOOKBACK, "float-lookback")):
        total = 0.0
        for code in range(1 << 5):
            path = bp.BernoulliPath(code, 5)
            total += bp.path_probability(P, path) * kind(P, case["S0"], case["K"], path)
        assert math.exp(-case["q"] * case["T"]) * total == pytest.approx(case["values"][tag], rel=1e-13)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted")
def test_reference_engine_accepts_our_callables():
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        import binpaths as R
    finally:
        sys.path.pop(0)
    inputs = R.MarketInputs(S0=100.0, K=100.0, q=0.05, sigma=0.2, T=1.0, N=8)
    P = R.TreeParams(dt=1 / 8, u=1.07, d=1 / 1.07, beta=1.0, up_probs=np.full(8, 0.52))
    ref_val = R.value_exact_serial(R.ValuationRequest(inputs=inputs, params=P, kind=bp.ASIAN_CALL))
    import oracle
    want = oracle.exact(8, 100.0, 100.0, 1.07, 1 / 1.07, 0.52, math.exp(-0.05), ["asian-call"])["asian-call"]
    assert ref_val == pytest.approx(want, rel=1e-13)
    # a reference PayoffKind member maps onto the same kernel bit
    assert bp.kind_bit(R.PayoffKind.ASIAN_PUT) == bp.kind_bit(bp.PayoffKind.ASIAN_PUT)


def test_mc_config_validation():
    for bad in (dict(R=0), dict(R=10, M=0), dict(R=10, seed=-1), dict(R=10, reps=0), dict(R=True)):
        with pytest.raises(bp.InvalidInput):
            bp.McConfig(**bad)
    inp = bp.MarketInputs(S0=20.0, K=100.0, q=0.06, sigma=3.0, T=1.0, N=12)
    req = bp.ValuationRequest(inputs=inp, params=bp.derive_crr(inp), kind=bp.PayoffKind.ASIAN_PUT)
    with pytest.raises(bp.InvalidInput):
        bp.estimate_basic(req, bp.McConfig(R=1))
    with pytest.raises(bp.InfeasibleAllocation):
        bp.estimate_partitioned(req, bp.McConfig(R=2, M=4))
    with pytest.raises(bp.InvalidWorkerCount):
        bp.estimate_partitioned(req, bp.McConfig(R=64, M=3))
    with pytest.raises(bp.InvalidInput):
        bp.estimate_shared(req, bp.McConfig(R=1, M=2))


def test_vectorised_partition_masses_are_bitwise_block_probability():
    from paper_1701_03512_b200 import paths
    rng = np.random.default_rng(3)
    for N in (5, 12, 40):
        P = bp.with_custom_probs(bp.MarketInputs(S0=1.0, K=1.0, q=0.0, sigma=0.2, T=1.0, N=N),
                                 rng.uniform(0.05, 0.95, N))
        for M in (1, 2, 3, 8, 16, 7):
            part = bp.make_partition(N, M)
            assert paths.partition_masses(P, part) == [bp.block_probability(P, part, m) for m in range(M)]
