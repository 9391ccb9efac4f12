"""A/B of library variants on the K1 headline shapes: alternating processes
(main, variant, main, variant, ...), each timing value_exact kernel_ms
(min and median of 20) for N=30 AC, FL, AC+FL and N=33 AC+FL.

  AB_ROUNDS=3 python tools/ab_k1.py <variant.so> [<variant.so> ...]
"""
import json
import os
import subprocess
import sys

CHILD = r'''
import os, sys, statistics, json
sys.path.insert(0, os.environ["REPO"])
import paper_1701_03512_b200 as bp
out = {}
for N, ks in ((30, [bp.ASIAN_CALL]), (30, [bp.FLOATING_LOOKBACK]), (30, [bp.ASIAN_CALL, bp.FLOATING_LOOKBACK]),
              (33, [bp.ASIAN_CALL, bp.FLOATING_LOOKBACK])):
    P = bp.classic_crr(N, 0.2, 0.05, 1.0)
    inp = bp.MarketInputs(S0=100.0, K=105.47846749285817, q=0.05, sigma=0.2, T=1.0, N=N)
    req = bp.ValuationRequest(inputs=inp, params=P, kind=ks[0], force_large=True)
    t = [bp.value_exact(req, kinds=ks, devices=[0]).kernel_ms * 1e3 for _ in range(25)][5:]
    out[f"N{N}:{'+'.join(k.tag for k in ks)}"] = (min(t), statistics.median(t))
print(json.dumps(out))
'''


def main():
    libs = [("main", None)] + [(os.path.basename(v), v) for v in sys.argv[1:]]
    rounds = int(os.environ.get("AB_ROUNDS", "3"))
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {tag: [] for tag, _ in libs}
    for _ in range(rounds):
        for tag, lib in libs:
            env = dict(os.environ, REPO=repo)
            env.pop("BINPATHS_LIB", None)
            if lib:
                env["BINPATHS_LIB"] = lib
            o = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            res[tag].append(json.loads(o.stdout.strip().splitlines()[-1]))
    for tag, runs in res.items():
        keys = runs[0].keys()
        print(tag, " ".join(f"{k}=min {min(r[k][0] for r in runs):.1f} med {sorted(r[k][1] for r in runs)[len(runs) // 2]:.1f}us"
                            for k in keys), flush=True)


if __name__ == "__main__":
    main()
