import os, sys, time, ctypes
sys.path.insert(0, os.getcwd())
import bench
import paper_1701_03512_b200 as bp
from paper_1701_03512_b200 import _native
from paper_1701_03512_b200.exact import tree_of
wl, crr = bench.workloads()
req, kinds, _ = bench.make_req(wl["config2"], crr)
for i in range(10):
    bp.value_exact(req, kinds=kinds, devices=[0])
N = 200
t0 = time.perf_counter()
for i in range(N):
    bp.value_exact(req, kinds=kinds, devices=[0])
t_api = (time.perf_counter() - t0) / N
tree, keep = tree_of(req)
arr = (ctypes.c_int * 1)(0)
res = _native.BpExactResult()
L = _native.lib()
t0 = time.perf_counter()
for i in range(N):
    L.bp_exact(ctypes.byref(tree), (1 << 4) | (1 << 5), 0, 1, arr, ctypes.byref(res))
t_c = (time.perf_counter() - t0) / N
print(f"value_exact {t_api*1e6:.1f} us, bare bp_exact via ctypes {t_c*1e6:.1f} us, kernel_ms {res.kernel_ms*1e3:.1f} us")
