"""Batched exact pricing (BASELINE configs[4]) vs reference goldens and the oracle."""
import math

import numpy as np
import pytest

import oracle
import paper_1701_03512_b200 as bp
from conftest import load_golden

pytestmark = pytest.mark.gpu


def config5_arrays(n=4096, seed=0):
    rng = np.random.default_rng(seed)
    S0 = rng.uniform(50, 150, n)
    m = rng.uniform(0.8, 1.2, n)
    K = m * S0
    sigma = rng.uniform(0.1, 0.5, n)
    r = rng.uniform(0.0, 0.08, n)
    T = rng.uniform(0.25, 3.0, n)
    return S0, K, sigma, r, T


def lattice(N, sigma, r, T):
    """classic CRR per option with math.exp (as the golden generator does)"""
    u = np.array([math.exp(s * math.sqrt(t / N)) for s, t in zip(sigma, T)])
    d = 1.0 / u
    p = np.array([(math.exp(rr * t / N) - dd) / (uu - dd) for rr, t, uu, dd in zip(r, T, u, d)])
    return u, d, p


def test_config5_full_batch_vs_reference_goldens():
    g = load_golden("exact_batch.json")
    N = g["N"]
    S0, K, sigma, r, T = config5_arrays()
    u, d, p = lattice(N, sigma, r, T)
    vals = bp.price_batch(N, S0, K, u, d, p, np.array([math.exp(-a * b) for a, b in zip(r, T)]), bp.ASIAN_CALL)
    assert vals.shape == (4096,)
    for o in g["options"]:
        i = o["index"]
        assert u[i] == o["u"] and p[i] == o["p"]
        assert vals[i] == pytest.approx(o["asian_call"], rel=1e-12), (i, vals[i], o["asian_call"])


@pytest.mark.parametrize("tag", ["asian-call", "asian-put", "float-lookback", "lookback-put", "euro-call", "euro-put"])
def test_batch_all_kinds_vs_oracle_and_single(tag):
    N = 18
    S0, K, sigma, r, T = config5_arrays(6, seed=5)
    u, d, p = lattice(N, sigma, r, T)
    disc = np.exp(-r * T)
    kind = bp.resolve_kind(tag)
    vals = bp.price_batch(N, S0, K, u, d, p, disc, kind)
    for i in range(6):
        want = oracle.exact(N, S0[i], K[i], u[i], d[i], p[i], disc[i], [tag], workers=8)[tag]
        assert vals[i] == pytest.approx(want, rel=1e-12, abs=1e-13), (tag, i, vals[i], want)


def test_batch_of_requests_matches_single_requests():
    reqs = []
    for K in (90.0, 100.0, 110.0):
        P = bp.classic_crr(20, 0.25, 0.04, 1.5)
        inp = bp.MarketInputs(S0=100.0, K=K, q=0.04, sigma=0.25, T=1.5, N=20)
        reqs.append(bp.ValuationRequest(inputs=inp, params=P, kind=bp.ASIAN_CALL))
    batch = bp.value_exact_batch(reqs)
    for v, req in zip(batch, reqs):
        assert v == pytest.approx(bp.value_exact_serial(req), rel=1e-12)
