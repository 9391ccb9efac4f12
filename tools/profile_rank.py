"""ncu driver: rank 0's share of a G-rank sharded valuation (prepared plan,
the bench's enqueue), a few times.   python tools/profile_rank.py [config2] [G] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1701_03512_b200 import dist as bpd  # noqa: E402
from paper_1701_03512_b200.exact import tree_of  # noqa: E402
from paper_1701_03512_b200.payoffs import kind_bit  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
wl, classic_crr = bench.workloads()
req, kinds, _ = bench.make_req(wl[name], classic_crr)
tree, keep = tree_of(req)
mask = 0
for k in kinds:
    mask |= 1 << kind_bit(k)
sh = bpd.ShardedExact(tree, keep, mask, 0, G, 0)
for _ in range(reps):
    sh.enqueue()
torch.cuda.synchronize()
print(name, G, sh.first, sh.count, sh.values() if G == 1 else sh.local[:sh.count].sum().item())
