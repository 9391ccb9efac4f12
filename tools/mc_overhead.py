"""Host overhead of one synchronous MC call (bp_mc_strata) at small sizes."""
import os
import sys
import time
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03512_b200 as bp  # noqa: E402
from paper_1701_03512_b200 import mc as bmc  # noqa: E402

P = bp.classic_crr(20, 0.2, 0.05, 1.0)
req = object.__new__(bp.ValuationRequest)
for f, v in dict(inputs=SimpleNamespace(S0=100.0, K=100.0, q=0.05, T=1.0, N=20), params=P, kind=bp.ASIAN_CALL,
                 workers=1, force_large=True).items():
    object.__setattr__(req, f, v)
for M_log2, R in ((0, 1024), (4, 256), (12, 64)):
    for _ in range(3):
        bmc._strata_stats(req, M_log2, [R] * (1 << M_log2), 0, 0, 1)
    ts, ks = [], []
    for _ in range(20):
        t0 = time.perf_counter()
        _, _, k = bmc._strata_stats(req, M_log2, [R] * (1 << M_log2), 0, 0, 1)
        ts.append(time.perf_counter() - t0)
        ks.append(k)
    ts.sort(); ks.sort()
    print(f"M=2^{M_log2} R_m={R}: wall {ts[10] * 1e3:.3f} ms, kernels {ks[10]:.3f} ms", flush=True)
    cfg = bp.McConfig(R=R << M_log2, M=1 << M_log2, seed=1)
    t0 = time.perf_counter()
    for _ in range(10):
        bp.estimate_partitioned(req, cfg)
    print(f"   estimate_partitioned: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms per call", flush=True)
