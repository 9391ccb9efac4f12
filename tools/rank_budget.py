"""Per-rank fixed-cost budget of the sharded exact valuation, measured on ONE
GPU, and the strong-scaling efficiency it predicts for G = 2, 4, 8 ranks.

For each G, rank 0's share of the canonical super-blocks (the largest share;
every rank's share is the same size for G | 64) is enqueued exactly as
bench.py's timed step does (prepared plan, CUDA-graph replay, L2 flushed,
CUDA events on the launch stream): K1 + K2 = the rank's device time.  The
exchange is one NCCL all_gather of the padded partials; here it runs in a
world-1 NCCL group (the call's own overhead, not the NVLink latency), and the
prediction is given for the measured world-1 time and for assumed 8-GPU
NVLink all_gather latencies.

  python tools/rank_budget.py [config2|config3] [unit_log2 ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    import bench
    from paper_1701_03512_b200 import dist as bpd
    from paper_1701_03512_b200.exact import tree_of
    from paper_1701_03512_b200.payoffs import kind_bit

    name = sys.argv[1] if len(sys.argv) > 1 else "config2"
    wl, classic_crr = bench.workloads()
    w = wl[name]
    req, kinds, _ = bench.make_req(w, classic_crr)
    tree, keep = tree_of(req)
    mask = 0
    for k in kinds:
        mask |= 1 << kind_bit(k)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1)
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")

    def timed(fn, n=30):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        out = []
        for _ in range(n):
            flush.fill_(1)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1))
        out.sort()
        return out[len(out) // 2]  # median

    res = {"workload": name, "paths": 2 ** w["N"], "ranks": {}}
    for G in (1, 2, 4, 8):
        sh = bpd.ShardedExact(tree, keep, mask, 0, G, 0)
        k_ms = timed(lambda: sh.enqueue(st))
        buf = torch.zeros_like(sh.local)
        out = torch.empty((buf.shape[0],) + tuple(buf.shape[1:]), dtype=buf.dtype, device=buf.device)
        x_ms = timed(lambda: dist.all_gather_into_tensor(out, buf))

        def step():  # the bench's timed step: this rank's launches, then the exchange (stream order)
            sh.enqueue(st)
            dist.all_gather_into_tensor(out, sh.local)

        s_ms = timed(step)
        res["ranks"][G] = {"superblocks": [sh.first, sh.count, sh.n_sb], "kernel_ms": k_ms,
                           "allgather_world1_ms": x_ms, "step_world1_ms": s_ms,
                           "exchange_in_step_ms": s_ms - k_ms}
        sh.close()
    t1 = res["ranks"][1]["kernel_ms"]
    res["predicted_efficiency"] = {}
    for G in (2, 4, 8):
        r = res["ranks"][G]
        res["predicted_efficiency"][G] = {
            f"exchange_{lab}": t1 / (G * (r["kernel_ms"] + x))
            for lab, x in (("world1_measured", r["allgather_world1_ms"]), ("10us", 0.010), ("20us", 0.020))}
        res["predicted_efficiency"][G]["kernel_only"] = t1 / (G * r["kernel_ms"])
        res["predicted_efficiency"][G]["step_world1_measured"] = res["ranks"][1]["step_world1_ms"] / (
            G * r["step_world1_ms"])
    res["unit_log2"] = os.environ.get("BINPATHS_UNIT_LOG2", "default (13)")
    print(json.dumps(res, indent=1))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
