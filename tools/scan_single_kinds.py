import sys, os
sys.path.insert(0, os.getcwd())
import paper_1701_03512_b200 as bp
for N in (30, 34):
    P = bp.classic_crr(N, 0.2, 0.05, 1.0)
    inp = bp.MarketInputs(S0=100.0, K=105.47846749285817, q=0.05, sigma=0.2, T=1.0, N=N)
    for ks in ([bp.ASIAN_CALL], [bp.FLOATING_LOOKBACK], [bp.ASIAN_CALL, bp.FLOATING_LOOKBACK]):
        req = bp.ValuationRequest(inputs=inp, params=P, kind=ks[0], force_large=True)
        ms = min(bp.value_exact(req, kinds=ks, devices=[0]).kernel_ms for _ in range(5))
        print(N, [k.tag for k in ks], f"{ms:.4f} ms", flush=True)
