"""A torchrun rank of the exact path's exchange, on CPU (gloo): launched by
tests/test_launch_cpu.py through paper_1701_03512_b200.launch.ensure_world,
the same launcher bench.py --gpus N uses.  Each rank takes its contiguous
range of the 64 canonical super-blocks, computes their partials with the
oracle (no GPU here), exchanges its padded buffer with one all_gather and
combines in ascending super-block order; every rank writes its values."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
from paper_1701_03512_b200 import dist as bpd  # noqa: E402

N, N_SB = 16, 64
U, P, S0, K, DISC = 1.04, 0.51, 100.0, 103.0, math.exp(-0.05)
KINDS = ["asian-call", "float-lookback"]


def partials(sbs):
    out = np.zeros((len(sbs), 6, 2))
    span = 1 << (N - 6)
    for i, sb in enumerate(sbs):
        v, _ = oracle.exact_range(N, S0, K, U, 1 / U, P, DISC, KINDS, sb * span, (sb + 1) * span, 1)
        out[i, 4, 0], out[i, 5, 0] = v["asian-call"], v["float-lookback"]
    return out


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    first, count = bpd.shard_range(N_SB, rank, world)
    local = torch.zeros((bpd.shard_rows(N_SB, world), 6, 2), dtype=torch.float64)
    local[:count] = torch.from_numpy(partials(range(first, first + count)))
    gathered = bpd.gather_partials(local, N_SB, world)
    vals = bpd.combine(bpd.unpad(gathered.numpy(), N_SB, world), (1 << 4) | (1 << 5))
    with open(os.path.join(sys.argv[1], f"rank{rank}.json"), "w") as f:
        json.dump({"rank": rank, "world": world, "first": first, "count": count, "values": vals}, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
