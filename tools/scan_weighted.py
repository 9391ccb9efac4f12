"""K1w (per-step probabilities, with_custom_probs) kernel time at N = 30."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1701_03512_b200 as bp  # noqa: E402

rng = np.random.default_rng(1)
for N, kinds in ((30, [bp.ASIAN_CALL]), (30, [bp.ASIAN_CALL, bp.FLOATING_LOOKBACK]), (32, [bp.ASIAN_CALL])):
    inp = bp.MarketInputs(S0=100.0, K=105.0, q=0.05, sigma=0.2, T=1.0, N=N)
    params = bp.with_custom_probs(inp, rng.uniform(0.45, 0.55, size=N))
    req = bp.ValuationRequest(inputs=inp, params=params, kind=kinds[0], force_large=True)
    res = [bp.value_exact(req, kinds=kinds) for _ in range(5)]
    print(f"N={N} kinds={len(kinds)} engine={res[-1].engine} ms={min(r.kernel_ms for r in res):.4f} "
          f"{res[-1].values}", flush=True)
