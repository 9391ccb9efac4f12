"""K1 kernel time (value_exact kernel_ms, best of 5) for a library variant:
N=30 Asian call, floating lookback, both fused (config 2 lattice) and N=36
Asian call (config 3).   BINPATHS_LIB=<variant.so> python tools/scan_k1.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03512_b200 as bp  # noqa: E402

tag = os.path.basename(os.environ.get("BINPATHS_LIB", "main"))
out = []
for N, sigma, r, T, K, ks in ((30, 0.2, 0.05, 1.0, 105.47846749285817, [bp.ASIAN_CALL]),
                              (30, 0.2, 0.05, 1.0, 105.47846749285817, [bp.FLOATING_LOOKBACK]),
                              (30, 0.2, 0.05, 1.0, 105.47846749285817, [bp.ASIAN_CALL, bp.FLOATING_LOOKBACK]),
                              (36, 0.3, 0.03, 2.0, 105.0, [bp.ASIAN_CALL])):
    P = bp.classic_crr(N, sigma, r, T)
    inp = bp.MarketInputs(S0=100.0, K=K, q=r, sigma=sigma, T=T, N=N)
    req = bp.ValuationRequest(inputs=inp, params=P, kind=ks[0], force_large=True)
    res = [bp.value_exact(req, kinds=ks, devices=[0]) for _ in range(5 if N < 36 else 3)]
    best = min(x.kernel_ms for x in res)
    out.append(f"N{N}:{'+'.join(k.tag for k in ks)}={best:.4f}ms")
print(tag, " ".join(out), flush=True)
