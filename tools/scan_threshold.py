"""Threshold-search engine (K8) timing: effective paths/s for N = 30..44."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1701_03512_b200 as bp  # noqa: E402

wl, crr = bench.workloads()
for name, N in (("config2", 30), ("config3", 36), ("config3", 40), ("config3", 44)):
    w = dict(wl[name], N=N)
    req, kinds, _ = bench.make_req(w, crr)
    ms = []
    for i in range(3):
        r = bp.value_exact(req, kinds=kinds, devices=[0], search=True)
        ms.append(r.kernel_ms)
    t = min(ms)
    print(f"{name} N={N} kinds={w['kinds']} search: {t:.3f} ms -> {2 ** N / t * 1e3:.3e} effective paths/s "
          f"values={r.values}", flush=True)
