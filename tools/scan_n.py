"""Fixed cost vs per-path cost of the exact engine: value_exact kernel_ms
(best of 5) over N for one kind at a time, config 2 lattice, and the
least-squares fit t = a + b * 2^N over N >= 28.

  python tools/scan_n.py [N_lo] [N_hi]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03512_b200 as bp  # noqa: E402

lo = int(sys.argv[1]) if len(sys.argv) > 1 else 24
hi = int(sys.argv[2]) if len(sys.argv) > 2 else 33
tag = os.path.basename(os.environ.get("BINPATHS_LIB", "main"))
for ks in ([bp.ASIAN_CALL], [bp.FLOATING_LOOKBACK], [bp.ASIAN_CALL, bp.FLOATING_LOOKBACK]):
    pts = []
    for N in range(lo, hi + 1):
        P = bp.classic_crr(N, 0.2, 0.05, 1.0)
        inp = bp.MarketInputs(S0=100.0, K=105.47846749285817, q=0.05, sigma=0.2, T=1.0, N=N)
        req = bp.ValuationRequest(inputs=inp, params=P, kind=ks[0], force_large=True)
        best = min(bp.value_exact(req, kinds=ks, devices=[0]).kernel_ms for _ in range(5))
        pts.append((N, best))
    fit = [(2.0 ** N, t) for N, t in pts if N >= 28]
    n = len(fit)
    mx = sum(x for x, _ in fit) / n
    my = sum(y for _, y in fit) / n
    b = sum((x - mx) * (y - my) for x, y in fit) / sum((x - mx) ** 2 for x, _ in fit)
    a = my - b * mx
    name = "+".join(k.tag for k in ks)
    print(tag, name, " ".join(f"N{N}={t * 1e3:.1f}us" for N, t in pts),
          f"| fit N>=28: fixed {a * 1e3:.1f} us, marginal {1.0 / (b * 1e-3):.3e} paths/s", flush=True)
