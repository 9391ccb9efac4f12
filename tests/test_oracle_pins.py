"""Pin the CPU oracle before trusting it (CPU only).

The oracle (oracle/bp_oracle.c) must reproduce: the golden vectors generated
from the unmodified reference (tests/golden/*.json, tools/make_goldens.py),
the reference's hand-enumerated toy values (tests/test_exact.py:35-39 of the
reference), its brute-force identities, and the published Philox4x32-10
known-answer vectors (Salmon et al., Random123).
"""
import math

import numpy as np
import pytest

import oracle
from conftest import load_golden

ALL = ["euro-call", "euro-put", "asian-put", "lookback-put", "asian-call", "float-lookback"]


def test_toy_tree_known_answers():
    # N=2, u=2, d=0.5, p=0.5, S0=4, K=5, q=0 (reference tests/test_exact.py:28-39)
    v = oracle.exact(2, 4.0, 5.0, 2.0, 0.5, 0.5, 1.0, ALL)
    assert v["euro-put"] == pytest.approx(1.5, abs=1e-12)
    assert v["asian-put"] == pytest.approx(1.375, abs=1e-12)
    assert v["lookback-put"] == pytest.approx(2.0, abs=1e-12)
    assert v["euro-call"] == pytest.approx(2.75, abs=1e-12)


def test_small_goldens_every_kind_every_case():
    g = load_golden("exact_small.json")
    for case in g["cases"]:
        N = case["N"]
        v = oracle.exact(N, case["S0"], case["K"], case["u"], case["d"], np.array(case["up_probs"]),
                         math.exp(-case["q"] * case["T"]), ALL)
        for k in ALL:
            want = case["values"][k]
            assert v[k] == pytest.approx(want, rel=1e-13, abs=1e-13), (case["tag"], k)
        # the sign-flip / two-run routes equal the callable route
        assert case["route_asian_call"] == pytest.approx(case["values"]["asian-call"], rel=1e-14, abs=1e-14)
        assert case["route_float_lookback"] == pytest.approx(case["values"]["float-lookback"], rel=1e-13, abs=1e-13)


def test_medium_goldens_and_worker_invariance():
    g = load_golden("exact_small.json")
    for case in g["medium"][:3]:
        N = case["N"]
        for workers in (1, 3, 8):
            v = oracle.exact(N, case["S0"], case["K"], case["u"], case["d"], case["p"],
                             math.exp(-case["q"] * case["T"]), ALL, workers=workers)
            for k in ALL:
                assert v[k] == pytest.approx(case["values"][k], rel=1e-12), (case["tag"], k, workers)


def test_config1_golden():
    g = load_golden("exact_config1.json")
    v = oracle.exact(20, 100.0, 100.0, g["u"], g["d"], g["p"], math.exp(-0.05),
                     ["asian-call", "float-lookback", "asian-put", "lookback-put"], workers=8)
    assert v["asian-call"] == pytest.approx(g["asian_call"], rel=1e-13)
    assert v["float-lookback"] == pytest.approx(g["float_lookback"], rel=1e-13)
    assert v["asian-put"] == pytest.approx(g["asian_put"], rel=1e-13)
    assert v["lookback-put"] == pytest.approx(g["fixed_lookback_put"], rel=1e-12)


def test_up_count_mass_is_binomial():
    # reference tests/test_paths.py:74-85: mass by up count = binom pmf
    N = 14
    vals, hist = oracle.exact(N, 1.0, 0.0, 1.1, 1 / 1.1, 0.3, 1.0, ["euro-call"], with_hist=True)
    assert [int(h) for h in hist] == [math.comb(N, h) for h in range(N + 1)]


def test_range_sum_adds_up_to_full_enumeration():
    g = load_golden("exact_config1.json")
    disc = math.exp(-0.05)
    full = oracle.exact(20, 100.0, 100.0, g["u"], g["d"], g["p"], disc, ["asian-call"], workers=4)
    a, na = oracle.exact_range(20, 100.0, 100.0, g["u"], g["d"], g["p"], disc, ["asian-call"], 0, 1 << 19, 4)
    b, nb = oracle.exact_range(20, 100.0, 100.0, g["u"], g["d"], g["p"], disc, ["asian-call"], 1 << 19, 1 << 20, 4)
    assert na + nb == 1 << 20
    assert a["asian-call"] + b["asian-call"] == pytest.approx(full["asian-call"], rel=1e-13)


@pytest.mark.parametrize("ctr,key,want", [
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
])
def test_philox_known_answers(ctr, key, want):
    assert oracle.philox4x32_10(ctr, key) == want


def test_mc_oracle_single_stratum_equals_basic_and_is_unbiased():
    g = load_golden("mc_reference.json")
    study = g["studies"][0]  # DESK tree, asian-put, N=12 (beta-CRR)
    from paper_1701_03512_b200 import MarketInputs, derive_crr
    inp = MarketInputs(S0=20.0, K=100.0, q=0.06, sigma=3.0, T=1.0, N=12)
    P = derive_crr(inp)
    reps = 200
    th, sse = oracle.mc_strata(12, 20.0, 100.0, P.u, P.d, P.up_probs, "asian-put", 0, [512], 31, 0, reps)
    disc = math.exp(-0.06)
    vals = disc * th[:, 0]
    se = vals.std(ddof=1) / math.sqrt(reps)
    assert abs(vals.mean() - study["exact"]) <= 4 * se
    # variance estimate calibrated against the empirical spread (20 %, test_mc.py:317-325)
    mean_var = np.mean(disc * disc * sse[:, 0] / 512 ** 2)
    assert mean_var == pytest.approx(vals.var(ddof=1), rel=0.25)


# ---------------------------------------------------------------------------
# The sampler (csrc/bp_mc_kernels.cu header; replaces sample_bits, mc.py:98-100)
def test_sampler_host_view_matches_oracle_bits():
    """PhiloxStream.bits (host view of the engine's stream) and the oracle's
    step-by-step restatement of the sampler give the same bits, for steps in
    both 32-step groups, forced steps (p = 1), p = 0, odd and even draws (the
    two halves of a pair block) and enough draws for first and later ties."""
    import paper_1701_03512_b200 as bp
    rng = np.random.default_rng(5)
    for N in (1, 7, 32, 33, 52, 64):
        probs = rng.uniform(0.0, 1.0, N)
        probs[::5] = 0.5 + 2.0 ** -20  # low threshold bits set: the tie words matter
        if N > 3:
            probs[1], probs[3] = 1.0, 0.0
        for stream, rep in ((0, 0), (11, 3)):
            host = bp.mc_stream(1234567890123, stream, rep)
            for draw in range(200):
                want = oracle.mc_bits(N, 0, probs, 1234567890123, stream, rep, draw)
                got = host.bits(probs)
                assert np.array_equal(got, want), (N, stream, rep, draw)


def test_sampler_frequencies_match_the_thresholds():
    """Each step is Bernoulli(floor(p 2^32) / 2^32): up-frequencies over 2^16
    draws stay within 5 sigma of p, including a threshold of 2^-8 + 2^-9 (the
    tie words carry half its mass) and one below 2^-8 (all of it)."""
    probs = np.array([0.5, 0.5077, 2.0 ** -8 + 2.0 ** -9, 2.0 ** -10, 0.999, 0.25, 1.0 - 2.0 ** -9, 0.75] * 5)
    N, R = probs.shape[0], 1 << 16
    ups = np.zeros(N)
    for draw in range(R):
        ups += oracle.mc_bits(N, 0, probs, 99, 2, 1, draw)
    sigma = np.sqrt(probs * (1 - probs) / R)
    assert np.all(np.abs(ups / R - probs) <= 5 * sigma), (ups / R - probs) / sigma
