"""Time the public API end to end (host inputs -> value back) for config 2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1701_03512_b200 as bp  # noqa: E402

wl, crr = bench.workloads()
req, kinds, _ = bench.make_req(wl["config2"], crr)
ts = []
for i in range(200):
    t0 = time.perf_counter()
    r = bp.value_exact(req, kinds=kinds, devices=[0])
    ts.append(time.perf_counter() - t0)
ts = sorted(ts[20:])
print(f"e2e median {ts[len(ts) // 2] * 1e3:.3f} ms  min {ts[0] * 1e3:.3f} ms  kernel {r.kernel_ms:.3f} ms")
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for i in range(20):
    bp.value_exact(req, kinds=kinds, devices=[0])
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
