"""Exact valuations beyond the BASELINE sizes (N = 40, 44): the explicit leaf
engine K1 against the threshold-search engine K8 (independent algorithms, same
exact value), with kernel times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03512_b200 as bp  # noqa: E402

for N in (40, 44):
    P = bp.classic_crr(N, 0.3, 0.03, 2.0)
    inp = bp.MarketInputs(S0=100.0, K=105.0, q=0.03, sigma=0.3, T=2.0, N=N)
    req = bp.ValuationRequest(inputs=inp, params=P, kind=bp.ASIAN_CALL, force_large=True)
    a = bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK])
    b = bp.value_exact(req, kinds=[bp.ASIAN_CALL, bp.FLOATING_LOOKBACK], search=True)
    print(f"N={N} 2^N={2 ** N:.3e} paths: K1 {a.kernel_ms:.1f} ms ({2 ** N / a.kernel_ms * 1e3:.3e} paths/s, both payoffs) "
          f"{a.values} | K8 {b.kernel_ms:.2f} ms {b.values} | rel diff "
          f"{max(abs(a.values[k] - b.values[k]) / abs(b.values[k]) for k in a.values):.2e}", flush=True)
