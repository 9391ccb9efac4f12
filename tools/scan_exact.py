"""Scan exact-engine kernel time over N / params / kinds (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03512_b200 as bp  # noqa: E402

cases = [
    (30, 0.2, 0.05, 1.0, 105.478, ["asian-call"]),
    (30, 0.2, 0.05, 1.0, 105.478, ["float-lookback"]),
    (30, 0.2, 0.05, 1.0, 105.478, ["asian-call", "float-lookback"]),
    (32, 0.2, 0.05, 1.0, 105.478, ["asian-call"]),
    (32, 0.3, 0.03, 2.0, 105.0, ["asian-call"]),
    (33, 0.2, 0.05, 1.0, 105.478, ["asian-call"]),
    (34, 0.2, 0.05, 1.0, 105.478, ["asian-call"]),
    (35, 0.2, 0.05, 1.0, 105.478, ["asian-call"]),
    (36, 0.2, 0.05, 1.0, 105.478, ["asian-call"]),
    (36, 0.3, 0.03, 2.0, 105.0, ["asian-call"]),
]
for N, sigma, r, T, K, kinds in cases:
    P = bp.classic_crr(N, sigma, r, T)
    inp = bp.MarketInputs(S0=100.0, K=K, q=r, sigma=sigma, T=T, N=N)
    ks = [bp.resolve_kind(k) for k in kinds]
    req = bp.ValuationRequest(inputs=inp, params=P, kind=ks[0], force_large=True)
    ms = []
    for i in range(3):
        res = bp.value_exact(req, kinds=ks, devices=[0])
        ms.append(res.kernel_ms)
    best = min(ms)
    print(f"N={N} sigma={sigma} kinds={kinds} engine={res.engine} ms={best:.3f} "
          f"paths/s={2**N / best * 1e3:.3e} values={res.values}", flush=True)
