"""GPU Monte Carlo vs the CPU oracle (same Philox4x32-10 draws -> agreement to
rounding) and against exact values / the reference's statistics.

Bars (BASELINE.json north_star): stratified MC within 4 standard errors of
the exact value; variance-reduction ratio over basic MC consistent with the
reference's (tests/golden/mc_reference.json).
"""
import math

import numpy as np
import pytest

import oracle
import paper_1701_03512_b200 as bp
from conftest import load_golden

pytestmark = pytest.mark.gpu

DESK = dict(S0=20.0, K=100.0, q=0.06, sigma=3.0, T=1.0)


def desk_req(kind=bp.PayoffKind.ASIAN_PUT, N=12):
    inputs = bp.MarketInputs(N=N, **DESK)
    return bp.ValuationRequest(inputs=inputs, params=bp.derive_crr(inputs), kind=kind)


def classic_req(N, kind=bp.ASIAN_CALL, S0=100.0, K=100.0, r=0.05, sigma=0.2, T=1.0):
    from types import SimpleNamespace
    P = bp.classic_crr(N, sigma, r, T)
    inputs = SimpleNamespace(S0=S0, K=K, q=r, sigma=sigma, T=T, N=N) if N > 62 else \
        bp.MarketInputs(S0=S0, K=K, q=r, sigma=sigma, T=T, N=N)
    return _req(inputs, P, kind)


def _req(inputs, P, kind):
    req = object.__new__(bp.ValuationRequest)
    object.__setattr__(req, "inputs", inputs)
    object.__setattr__(req, "params", P)
    object.__setattr__(req, "kind", kind)
    object.__setattr__(req, "workers", 1)
    object.__setattr__(req, "force_large", True)
    return req


TAGS = ["euro-call", "euro-put", "asian-put", "lookback-put", "asian-call", "float-lookback"]


@pytest.mark.parametrize("tag", TAGS)
def test_strata_stats_match_oracle_draw_for_draw(tag):
    req = desk_req(bp.resolve_kind(tag))
    P = req.params
    r, M = 2, 4
    alloc = [300, 5000, 1, 0]
    theta, sse, _ = bp.mc._strata_stats(req, r, alloc, 1234, 3, 2)
    ot, os_ = oracle.mc_strata(12, DESK["S0"], DESK["K"], P.u, P.d, P.up_probs, tag, r, alloc, 1234, 3, 2)
    np.testing.assert_allclose(theta, ot, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(sse, os_, rtol=1e-10, atol=1e-9)
    assert theta[0, 3] == 0.0 and sse[0, 3] == 0.0


def test_shared_matches_oracle():
    req = desk_req()
    P = req.params
    masses = np.array([bp.block_probability(P, bp.make_partition(12, 8), m) for m in range(8)])
    est = [bp.estimate_shared(req, bp.McConfig(R=5000, M=8, seed=77), rep=k) for k in range(2)]
    oim, oisse, osm = oracle.mc_shared(12, DESK["S0"], DESK["K"], P.u, P.d, P.up_probs, "asian-put", 3, 5000,
                                       masses, 77, 0, 2)
    disc = math.exp(-DESK["q"] * DESK["T"])
    for k in range(2):
        assert est[k].value == pytest.approx(disc * oim[k], rel=1e-12)
        assert est[k].variance == pytest.approx(disc * disc * oisse[k] / 5000 ** 2, rel=1e-9)
        np.testing.assert_allclose([t for _, _, t in est[k].per_stratum], osm[k], rtol=1e-12)


def test_single_stratum_is_bitwise_basic():
    req = desk_req()
    for rep in range(3):
        base = bp.estimate_basic(req, bp.McConfig(R=256, seed=5), rep=rep)
        part = bp.estimate_partitioned(req, bp.McConfig(R=256, M=1, seed=5), rep=rep)
        eq = bp.estimate_partitioned_equal(req, bp.McConfig(R=256, M=1, seed=5), rep=rep)
        assert base.value == part.value == eq.value
        assert base.variance == part.variance == eq.variance


def test_run_repetitions_batched_equals_per_rep():
    req = desk_req()
    cfg = bp.McConfig(R=300, M=4, seed=9, reps=5)
    s = bp.run_repetitions(bp.estimate_partitioned, req, cfg)
    for k in range(5):
        assert s.estimates[k] == bp.estimate_partitioned(req, cfg, rep=k)


def test_full_stratification_recovers_exact_value():
    inputs = bp.MarketInputs(S0=5.0, K=10.0, q=0.06, sigma=0.50, T=1.0, N=4)
    req = bp.ValuationRequest(inputs=inputs, params=bp.derive_crr(inputs), kind=bp.PayoffKind.ASIAN_PUT)
    exact = bp.value_exact_serial(req)
    est = bp.estimate_partitioned(req, bp.McConfig(R=16, M=16, seed=0))
    assert est.variance == 0.0
    assert est.value == pytest.approx(exact, rel=1e-12)
    eq = bp.estimate_partitioned_equal(req, bp.McConfig(R=5, M=16, seed=0))
    assert eq.variance <= 1e-28 and eq.value == pytest.approx(exact, rel=1e-12) and eq.R_used == 80
    sh = bp.estimate_shared(req, bp.McConfig(R=8, M=16, seed=0))
    assert sh.variance <= 1e-28 and sh.value == pytest.approx(exact, rel=1e-12)


def test_zero_mass_strata_are_skipped():
    inputs = bp.MarketInputs(S0=2.0, K=1.0, q=0.05, sigma=0.0, T=1.0, N=8)
    params = bp.derive_crr(inputs)
    req = bp.ValuationRequest(inputs=inputs, params=params, kind=bp.PayoffKind.EUROPEAN_CALL)
    est = bp.estimate_partitioned(req, bp.McConfig(R=8, M=4, seed=0))
    assert [d for _, d, _ in est.per_stratum] == [0, 0, 0, 8]
    assert est.variance <= 1e-30
    assert est.value == pytest.approx(math.exp(-0.05) * (2.0 * params.u ** 8 - 1.0), rel=1e-13)


@pytest.mark.parametrize("N", [20, 30, 36])
def test_stratified_within_4se_of_exact(N):
    req = classic_req(N)
    exact = bp.value_exact(req, kinds=[bp.ASIAN_CALL]).values["asian-call"]
    est = bp.estimate_partitioned_equal(req, bp.McConfig(R=1 << 10, M=1 << 12, seed=11))
    assert abs(est.value - exact) <= 4 * est.std_error, (est.value, exact, est.std_error)
    b = bp.estimate_basic(req, bp.McConfig(R=1 << 22, seed=11))
    assert abs(b.value - exact) <= 4 * b.std_error


def test_unbiased_over_repetitions_all_kinds():
    reps = 400
    for kind in bp.PayoffKind:
        req = desk_req(kind)
        exact = bp.value_exact_serial(req)
        for est, cfg in [(bp.estimate_basic, bp.McConfig(R=128, seed=31, reps=reps)),
                         (bp.estimate_partitioned, bp.McConfig(R=128, M=4, seed=37, reps=reps)),
                         (bp.estimate_partitioned_equal, bp.McConfig(R=32, M=4, seed=41, reps=reps)),
                         (bp.estimate_shared, bp.McConfig(R=128, M=4, seed=43, reps=reps))]:
            s = bp.run_repetitions(est, req, cfg)
            se = s.values.std(ddof=1) / math.sqrt(reps)
            assert abs(s.mean_value - exact) <= 4.0 * se, (kind, est.__name__, s.mean_value, exact, se)


@pytest.mark.parametrize("N", [32, 62])
def test_variance_reduction_ratio_consistent_with_reference(N):
    g = load_golden("mc_reference.json")
    ref = next(s for s in g["studies"] if s.get("tree") == "classic" and s["N"] == N)
    req = classic_req(N)
    reps = 10
    R_total = ref["R_total"]
    b = bp.run_repetitions(bp.estimate_basic, req, bp.McConfig(R=R_total, seed=7, reps=reps))
    e = bp.run_repetitions(bp.estimate_partitioned_equal, req, bp.McConfig(R=R_total >> 12, M=4096, seed=7, reps=reps))
    ratio = b.mean_variance / e.mean_variance
    # per-rep variance estimates have relative noise ~ sqrt(2/R): the ratio of
    # 10-rep means is known to a few per cent; allow 15 %
    assert ratio == pytest.approx(ref["ratio_basic_over_equal"], rel=0.15), (ratio, ref["ratio_basic_over_equal"])
    assert b.mean_value == pytest.approx(ref["basic"]["mean_value"], abs=6 * math.sqrt(b.mean_variance))


def test_per_step_probabilities_and_N64_match_oracle():
    """Non-constant per-step probabilities (with_custom_probs, model.py:152-161)
    take the general sampler path; N = 64 (config 4 depth, beyond the
    reference's MAX_DEPTH) runs through the same stream layout."""
    from types import SimpleNamespace
    rng = np.random.default_rng(3)
    inputs = bp.MarketInputs(S0=50.0, K=52.0, q=0.03, sigma=0.4, T=1.0, N=14)
    params = bp.with_custom_probs(inputs, rng.uniform(0.2, 0.8, size=14))
    for tag in ("asian-call", "float-lookback", "lookback-put"):
        req = bp.ValuationRequest(inputs=inputs, params=params, kind=bp.resolve_kind(tag))
        draws = [700, 3, 5000, 1]
        theta, sse, _ = bp.mc._strata_stats(req, 2, draws, 99, 0, 1)
        ot, os_ = oracle.mc_strata(14, 50.0, 52.0, params.u, params.d, params.up_probs, tag, 2, draws, 99, 0, 1)
        np.testing.assert_allclose(theta, ot, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(sse, os_, rtol=1e-9, atol=1e-9)
    req64 = classic_req(64)
    P = req64.params
    theta, sse, _ = bp.mc._strata_stats(req64, 3, [2000] * 8, 5, 1, 1)
    ot, os_ = oracle.mc_strata(64, 100.0, 100.0, P.u, P.d, P.up_probs, "asian-call", 3, [2000] * 8, 5, 1, 1)
    np.testing.assert_allclose(theta, ot, rtol=1e-12)
    np.testing.assert_allclose(sse, os_, rtol=1e-9)


def test_sigma_zero_all_up_paths():
    """p == 1 exactly (sigma = 0, model.py:128-132): every draw is the all-up path."""
    inputs = bp.MarketInputs(S0=2.0, K=1.0, q=0.05, sigma=0.0, T=1.0, N=8)
    params = bp.derive_crr(inputs)
    req = bp.ValuationRequest(inputs=inputs, params=params, kind=bp.PayoffKind.EUROPEAN_CALL)
    est = bp.estimate_basic(req, bp.McConfig(R=64, seed=1))
    assert est.variance == 0.0
    assert est.value == pytest.approx(math.exp(-0.05) * (2.0 * params.u ** 8 - 1.0), rel=1e-13)


def test_sampler_later_ties_match_oracle_at_depth():
    """2^20 draws of 64 (62) stream-decided steps: about 7000 draws have a
    second tie in a group and ~300 a third, so the pair block, the overflow
    blocks and the per-step tie thresholds (general path) are all exercised;
    one wrong bit in one draw would move theta by ~1e-7 relative."""
    R = 1 << 20
    req64 = classic_req(64)
    P = req64.params
    theta, sse, _ = bp.mc._strata_stats(req64, 0, [R], 17, 0, 1)
    ot, os_ = oracle.mc_strata(64, 100.0, 100.0, P.u, P.d, P.up_probs, "asian-call", 0, [R], 17, 0, 1)
    np.testing.assert_allclose(theta, ot, rtol=1e-12)
    np.testing.assert_allclose(sse, os_, rtol=1e-9)
    rng = np.random.default_rng(8)
    inputs = bp.MarketInputs(S0=50.0, K=52.0, q=0.03, sigma=0.4, T=1.0, N=62)
    params = bp.with_custom_probs(inputs, rng.uniform(0.05, 0.95, size=62))
    req = bp.ValuationRequest(inputs=inputs, params=params, kind=bp.resolve_kind("float-lookback"), force_large=True)
    theta, sse, _ = bp.mc._strata_stats(req, 0, [R // 4], 23, 2, 1)
    ot, os_ = oracle.mc_strata(62, 50.0, 52.0, params.u, params.d, params.up_probs, "float-lookback", 0, [R // 4],
                               23, 2, 1)
    np.testing.assert_allclose(theta, ot, rtol=1e-12)
    np.testing.assert_allclose(sse, os_, rtol=1e-9)


def test_forced_and_impossible_steps_in_the_suffix_match_oracle():
    """Per-step probabilities with p = 1 (forced up, not drawn) and p = 0 steps
    inside the stream-decided suffix, including the first suffix step, in both
    32-step groups (N = 40, r = 2), and a constant-p tree whose first suffix
    step is forced (the kernel then takes the general path)."""
    N, r = 40, 2
    rng = np.random.default_rng(12)
    probs = rng.uniform(0.1, 0.9, size=N)
    probs[[r, 7, 33, 39]] = 1.0
    probs[[5, 20, 36]] = 0.0
    inputs = bp.MarketInputs(S0=50.0, K=48.0, q=0.02, sigma=0.3, T=1.0, N=N)
    base = bp.derive_crr(inputs)

    def tree(p):  # with_custom_probs keeps to the open interval; the engine takes [0, 1]
        return bp.TreeParams(dt=base.dt, u=base.u, d=base.d, beta=base.beta, up_probs=p)

    params = tree(probs)
    draws = [3000, 1, 4097, 500]
    for tag in ("asian-call", "lookback-put"):
        req = bp.ValuationRequest(inputs=inputs, params=params, kind=bp.resolve_kind(tag), force_large=True)
        theta, sse, _ = bp.mc._strata_stats(req, r, draws, 31, 0, 2)
        ot, os_ = oracle.mc_strata(N, 50.0, 48.0, params.u, params.d, params.up_probs, tag, r, draws, 31, 0, 2)
        np.testing.assert_allclose(theta, ot, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(sse, os_, rtol=1e-9, atol=1e-9)
    const = np.full(N, 0.55)
    const[r] = 1.0
    params = tree(const)
    req = bp.ValuationRequest(inputs=inputs, params=params, kind=bp.ASIAN_CALL, force_large=True)
    theta, sse, _ = bp.mc._strata_stats(req, r, draws, 32, 1, 1)
    ot, os_ = oracle.mc_strata(N, 50.0, 48.0, params.u, params.d, params.up_probs, "asian-call", r, draws, 32, 1, 1)
    np.testing.assert_allclose(theta, ot, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(sse, os_, rtol=1e-9, atol=1e-9)
