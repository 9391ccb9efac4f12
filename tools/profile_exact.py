"""Small driver for ncu: runs a few exact valuations of one BASELINE workload.

  python tools/profile_exact.py [config2|config3|N30ac] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1701_03512_b200 as bp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl, classic_crr = bench.workloads()
if name == "N30ac":
    w = dict(wl["config2"], kinds=["asian-call"])
elif name == "N30fl":
    w = dict(wl["config2"], kinds=["float-lookback"])
elif name == "N32ac":
    w = dict(wl["config2"], N=32, kinds=["asian-call"])
else:
    w = wl[name]
req, kinds, _ = bench.make_req(w, classic_crr)
for i in range(reps):
    r = bp.value_exact(req, kinds=kinds, devices=[0])
    print(name, r.values, f"{r.kernel_ms:.3f} ms", flush=True)
