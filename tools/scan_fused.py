"""Kernel time of the exact engine for variant scans: the fused config-2
kernel (Asian call + floating lookback) over N, and the config-3 Asian call.
  BINPATHS_LIB=<variant.so> python tools/scan_fused.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03512_b200 as bp  # noqa: E402

tag = os.path.basename(os.environ.get("BINPATHS_LIB", "main"))
cases = [(N, 0.2, 0.05, 1.0, 105.47846749285817, [bp.ASIAN_CALL, bp.FLOATING_LOOKBACK]) for N in (30, 32, 34)]
cases.append((36, 0.3, 0.03, 2.0, 105.0, [bp.ASIAN_CALL]))
for N, sigma, r, T, K, ks in cases:
    P = bp.classic_crr(N, sigma, r, T)
    inp = bp.MarketInputs(S0=100.0, K=K, q=r, sigma=sigma, T=T, N=N)
    req = bp.ValuationRequest(inputs=inp, params=P, kind=ks[0], force_large=True)
    res = [bp.value_exact(req, kinds=ks, devices=[0]) for _ in range(5 if N < 36 else 3)]
    best = min(x.kernel_ms for x in res)
    vals = " ".join(f"{k}={v:.15g}" for k, v in res[-1].values.items())
    print(f"{tag} unit={os.environ.get('BINPATHS_UNIT_LOG2', '13')} N={N} kinds={len(ks)} ms={best:.4f} "
          f"paths/s={2**N / best * 1e3:.3e} {vals}", flush=True)
