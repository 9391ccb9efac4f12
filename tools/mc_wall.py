import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
from types import SimpleNamespace
import paper_1701_03512_b200 as bp
from paper_1701_03512_b200 import mc as bmc
N, k, R_m = 64, 12, 65536
P = bp.classic_crr(N, 0.2, 0.05, 1.0)
req = object.__new__(bp.ValuationRequest)
for f, v in dict(inputs=SimpleNamespace(S0=100.0, K=100.0, q=0.05, sigma=0.2, T=1.0, N=N), params=P,
                 kind=bp.ASIAN_CALL, workers=1, force_large=True, devices=[0]).items():
    object.__setattr__(req, f, v)
draws = [R_m] * (1 << k)
for i in range(3): bmc._strata_stats(req, k, draws, 0, 0, 1)
ts = []
for i in range(10):
    t0 = time.perf_counter(); _, _, ms = bmc._strata_stats(req, k, draws, 0, 0, 1); ts.append((time.perf_counter() - t0) * 1e3)
print("strata_stats wall min %.3f ms median %.3f ms, kernel %.3f ms" % (min(ts), sorted(ts)[5], ms))
ts = []
for i in range(5):
    t0 = time.perf_counter(); e = bp.estimate_partitioned_equal(req, bp.McConfig(R=R_m, M=1 << k, seed=0)); ts.append((time.perf_counter() - t0) * 1e3)
print("estimate_partitioned_equal wall min %.3f ms" % min(ts))
# config 5: the batched exact call
import math
n, Nb = 4096, 24
rng = np.random.default_rng(0)
S0 = rng.uniform(50, 150, n); m = rng.uniform(0.8, 1.2, n); K = m * S0
sigma = rng.uniform(0.1, 0.5, n); r = rng.uniform(0.0, 0.08, n); T = rng.uniform(0.25, 3.0, n)
u = np.exp(sigma * np.sqrt(T / Nb)); d = 1.0 / u
p = (np.exp(r * T / Nb) - d) / (u - d); disc = np.exp(-r * T)
for i in range(2): bp.price_batch(Nb, S0, K, u, d, p, disc, bp.ASIAN_CALL, device=0, with_time=True)
ts = []
for i in range(5):
    t0 = time.perf_counter(); vals, kms = bp.price_batch(Nb, S0, K, u, d, p, disc, bp.ASIAN_CALL, device=0, with_time=True); ts.append((time.perf_counter() - t0) * 1e3)
print("price_batch wall min %.3f ms, kernel %.3f ms" % (min(ts), kms))
