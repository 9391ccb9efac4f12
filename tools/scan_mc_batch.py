"""Time BASELINE configs[3] (stratified MC, N=64) and configs[4] (batched exact, 4096 x N=24)."""
import os
import sys
import time
from types import SimpleNamespace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03512_b200 as bp  # noqa: E402
from paper_1701_03512_b200 import mc as bmc  # noqa: E402


def mc_config4(R_m=65536, k=12, N=64):
    P = bp.classic_crr(N, 0.2, 0.05, 1.0)
    inputs = SimpleNamespace(S0=100.0, K=100.0, q=0.05, sigma=0.2, T=1.0, N=N)
    req = object.__new__(bp.ValuationRequest)
    for f, v in dict(inputs=inputs, params=P, kind=bp.ASIAN_CALL, workers=1, force_large=True).items():
        object.__setattr__(req, f, v)
    for i in range(2):
        t0 = time.perf_counter()
        theta, sse, ms = bmc._strata_stats(req, k, [R_m] * (1 << k), 0, 0, 1)
        wall = time.perf_counter() - t0
    draws = R_m << k
    print(f"config4 stratified N={N} k={k} R_m={R_m}: kernel {ms:.2f} ms -> {draws / ms * 1e3:.3e} draws/s "
          f"(wall {wall * 1e3:.1f} ms)", flush=True)
    t0 = time.perf_counter()
    e = bp.estimate_partitioned_equal(req, bp.McConfig(R=R_m, M=1 << k, seed=0))
    b = bp.estimate_basic(req, bp.McConfig(R=draws, seed=0))
    print(f"  pmc-equal {e.value:.6f} se {e.std_error:.2e}; basic {b.value:.6f} se {b.std_error:.2e}; "
          f"variance ratio {b.variance / e.variance:.3f}; wall {time.perf_counter() - t0:.2f} s", flush=True)


def batch_config5(n=4096, N=24):
    rng = np.random.default_rng(0)
    S0 = rng.uniform(50, 150, n); m = rng.uniform(0.8, 1.2, n); K = m * S0
    sigma = rng.uniform(0.1, 0.5, n); r = rng.uniform(0.0, 0.08, n); T = rng.uniform(0.25, 3.0, n)
    u = np.exp(sigma * np.sqrt(T / N)); d = 1 / u; p = (np.exp(r * T / N) - d) / (u - d)
    for i in range(2):
        vals, ms = bp.price_batch(N, S0, K, u, d, p, np.exp(-r * T), bp.ASIAN_CALL, with_time=True)
    paths = n * (1 << N)
    print(f"config5 batch {n} x N={N}: kernel {ms:.2f} ms -> {paths / ms * 1e3:.3e} paths/s", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["mc", "batch"]
    if "mc" in which:
        mc_config4()
    if "batch" in which:
        batch_config5()
