"""The paper's published Monte Carlo studies (Tables 3-5, N = 32,
beta-CRR desk tree S0=20, K=100, q=6%, sigma=3, T=1), reproduced by the GPU
estimators: mean of the per-repetition variance estimates over 1000
repetitions vs the published variance estimates (single runs rounded to 3
decimals, hence the tolerances), and the published exact values 82.115 /
93.196 within 4 standard errors of the repetition mean.
"""
import math
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import paper_tables as pt  # noqa: E402
import paper_1701_03512_b200 as bp  # noqa: E402

pytestmark = pytest.mark.gpu
REPS = 1000


@pytest.fixture(scope="module")
def study():
    return pt.study(REPS)


def _check(ours, pub, rel, abs_=0.0015):
    for k, v in pub.items():
        assert abs(ours[k] - v) <= max(rel * v, abs_), (k, ours[k], v)


def test_table3_basic_mc_variance(study):
    _check(study["table3_basic_var_asian"], pt.PUBLISHED["table3_basic_var_asian"], rel=0.12)
    _check(study["table3_basic_var_lookback"], pt.PUBLISHED["table3_basic_var_lookback"], rel=0.25)


def test_table4_partitioned_variance_shrinks_like_the_paper(study):
    _check(study["table4_partitioned_prop_var_asian"], pt.PUBLISHED["table4_partitioned_prop_var_asian"], rel=0.12)
    _check(study["table4_partitioned_prop_var_lookback"], pt.PUBLISHED["table4_partitioned_prop_var_lookback"],
           rel=0.15)


def test_table5_shared_sample_and_partitioned_ordering(study):
    _check(study["table5_shared_var_asian"], pt.PUBLISHED["table5_shared_var_asian"], rel=0.10)
    part, shared = study["table5_partitioned_var_asian"], study["table5_shared_var_asian"]
    # Theorem 1: partitioned (R per stratum) <= shared sample
    for M in part:
        assert part[M] <= shared[M] * 1.02, (M, part[M], shared[M])
    # The published partitioned column is ONE run per cell.  Each cell is
    # placed in the distribution of our 1000 single-run variance estimates:
    # M = 1, 4, 8, 32, 64 lie inside its central 99 % (within the published
    # rounding to 3 decimals); the published M = 2
    # (0.220) and M = 16 (0.005) lie outside it (M = 2 above, M = 16 below; the
    # bands are in profiles/r2_paper_tables_1000reps.json and DESIGN.md 3).
    # The test pins exactly that: any other cell leaving the band fails.
    pub = pt.PUBLISHED["table5_partitioned_var_asian"]
    outside = {}
    for M, v in pub.items():
        lo, hi = study["table5_partitioned_var_asian_q"][M]
        # the published value is rounded to 3 decimals: it stands for [v - 5e-4, v + 5e-4]
        if v + 5e-4 < lo or v - 5e-4 > hi:
            outside[M] = "above" if v - 5e-4 > hi else "below"
    assert outside == {2: "above", 16: "below"}, outside
    # where the published run sits inside the band, our mean tracks it within 25 %
    _check({M: part[M] for M in (1, 4, 8, 32, 64)}, {M: pub[M] for M in (1, 4, 8, 32, 64)}, rel=0.25)


def test_published_exact_values_within_4se():
    for kind, target in ((bp.PayoffKind.ASIAN_PUT, 82.115), (bp.PayoffKind.FIXED_LOOKBACK_PUT, 93.196)):
        s = bp.run_repetitions(bp.estimate_partitioned, pt.desk(kind), bp.McConfig(R=1 << 12, M=16, seed=7,
                                                                                   reps=REPS))
        se = s.values.std(ddof=1) / math.sqrt(REPS)
        assert abs(s.mean_value - target) <= 4 * se + 5e-4, (kind, s.mean_value, target, se)
