"""Benchmark: exact-enumeration paths/s on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload config2|config3|config1]

One step = one exact valuation of the workload's tree: every one of the 2^N
paths evaluated (both payoffs of config 2 in one pass), the per-rank
super-block partials reduced, exchanged (NCCL all_gather when N > 1) and
combined.  Default workload = BASELINE configs[1] (N = 30, Asian call +
floating lookback, K from default_rng(0)); config 3 (N = 36 Asian call) is
measured in the same run and reported under "config3".

N > 1 runs under torchrun, one rank per GPU; each rank owns a contiguous
range of the 64 canonical super-blocks ("scaling": "weak" is NOT claimed --
the total work is fixed, so scaling is "strong").

--impl reference times the reference algorithm on the host CPU: the C
restatement in oracle/ (the reference is pure Python and cannot be compiled;
its own numpy engine was measured at 1.3e7 paths/s on 8 cores, BASELINE.md
§3), on a bounded sample of the same workload with every host thread.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W_OPS = {"asian-call": 3, "float-lookback": 3}  # FP64-pipe ops per path per payoff
# one metric string for both arms (ours and --impl reference)
METRIC = "exact-enumeration paths/sec (N=30 two payoffs in one pass; N=36 under config3)"


def workloads():
    import numpy as np
    from paper_1701_03512_b200 import classic_crr

    K2 = float(np.random.default_rng(0).uniform(80, 120))
    return {
        "config1": dict(N=20, S0=100.0, K=100.0, r=0.05, sigma=0.2, T=1.0, kinds=["asian-call"]),
        "config2": dict(N=30, S0=100.0, K=K2, r=0.05, sigma=0.2, T=1.0, kinds=["asian-call", "float-lookback"]),
        "config3": dict(N=36, S0=100.0, K=105.0, r=0.03, sigma=0.3, T=2.0, kinds=["asian-call"]),
    }, classic_crr


def workload_config(name, w):
    """The workload keys both arms report (same config for the driver's ratio)."""
    return {"workload": name, "N": w["N"], "payoffs": w["kinds"], "K": w["K"], "S0": w["S0"], "r": w["r"],
            "sigma": w["sigma"], "T": w["T"]}


def make_req(w, classic_crr):
    import paper_1701_03512_b200 as bp
    P = classic_crr(w["N"], w["sigma"], w["r"], w["T"])
    inputs = bp.MarketInputs(S0=w["S0"], K=w["K"], q=w["r"], sigma=w["sigma"], T=w["T"], N=w["N"])
    kinds = [bp.resolve_kind(k) for k in w["kinds"]]
    return bp.ValuationRequest(inputs=inputs, params=P, kind=kinds[0], force_large=True), kinds, P


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def cpu_baseline(w, classic_crr, budget_s=12.0):
    """Reference algorithm (oracle/ C restatement) on every host thread, on a
    bounded contiguous sample of the workload's path codes."""
    import oracle
    P = classic_crr(w["N"], w["sigma"], w["r"], w["T"])
    threads = os.cpu_count() or 1
    disc = math.exp(-w["r"] * w["T"])
    n = 1 << 16
    elapsed = 0.0
    while True:
        t0 = time.perf_counter()
        _, paths = oracle.exact_range(w["N"], w["S0"], w["K"], P.u, P.d, P.up_probs[0], disc, w["kinds"], 0, n,
                                      threads)
        elapsed = time.perf_counter() - t0
        if elapsed * 4 > budget_s or n >= (1 << w["N"]):
            break
        n <<= 2
    return {"value": paths / elapsed, "unit": "paths/s", "cores": threads, "kind": "port",
            "sample": f"{paths} of 2^{w['N']} paths (codes [0, {paths})), {'+'.join(w['kinds'])} in one pass, "
                      f"{elapsed:.2f} s wall, oracle/bp_oracle.c (per-path walk as exact.py:83-100)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl, classic_crr = workloads()
    w = wl[args.workload]
    steps = []
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline(w, classic_crr, budget_s=4.0 if i >= args.warmup else 1.0)
        if i >= args.warmup:
            steps.append(cb)
    v = statistics.median(s["value"] for s in steps)
    total = 1 << w["N"]
    line = {"metric": METRIC, "value": v, "unit": "paths/s",
            "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / v * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {**workload_config(args.workload, w), "parallelism": f"{os.cpu_count()} host threads"},
            "cpu_baseline": {**steps[-1], "value": v},
            "e2e": {"value": v, "unit": "paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def time_workload(w, classic_crr, steps, warmup, rank, world, dev, group):
    """Device-timed steps (CUDA events on the launch stream), L2 flushed
    between steps; returns (ms list, values, sharder)."""
    import torch
    import torch.distributed as dist
    from paper_1701_03512_b200 import dist as bpd
    from paper_1701_03512_b200.exact import tree_of
    from paper_1701_03512_b200.payoffs import kind_bit

    req, kinds, P = make_req(w, classic_crr)
    tree, keep = tree_of(req)
    mask = 0
    for k in kinds:
        mask |= 1 << kind_bit(k)
    sh = bpd.ShardedExact(tree, keep, mask, rank, world, dev)
    st = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")  # > 126 MB L2
    for _ in range(warmup):
        sh.enqueue(st)
        sh.exchange(group)
    torch.cuda.synchronize(dev)
    times = []
    for _ in range(steps):
        flush.fill_(1)
        if world > 1:
            dist.barrier(group=group)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sh.enqueue(st)
        sh.exchange(group)
        e1.record(st)
        torch.cuda.synchronize(dev)
        times.append(e0.elapsed_time(e1))
    vals = sh.values()
    return times, vals, sh, req, kinds


def e2e_seconds(bp, req, kinds, args, warmup, rank, world, dev, group):
    """Median wall seconds of one public-API valuation (host request in,
    Python floats out), max over ranks.  N = 1: value_exact (C ABI, one
    synchronous call); N > 1: value_exact_distributed on every rank (this
    rank's super-blocks, the NCCL all_gather, the host combine)."""
    import torch
    import torch.distributed as dist
    from paper_1701_03512_b200 import dist as bpd

    ts = []
    for i in range(warmup + args.steps):
        if world > 1:
            dist.barrier(group=group)
        t0 = time.perf_counter()
        if world == 1:
            bp.value_exact(req, kinds=kinds, devices=[dev])
        else:
            bpd.value_exact_distributed(req, kinds, rank=rank, world=world, device=dev, group=group)
        dt = time.perf_counter() - t0
        if i >= warmup:
            ts.append(dt)
    med = statistics.median(ts)
    if world > 1:
        t = torch.tensor([med], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        med = float(t.item())
        return med, "paper_1701_03512_b200.dist.value_exact_distributed(req, kinds, rank, world) on every rank"
    return med, "paper_1701_03512_b200.value_exact(req, kinds) -> bp_exact (C ABI)"


def kernel_share(w, classic_crr, dev, reps=5):
    """Duration of the dominant kernel alone (the leaf kernel + its reduce are
    what one super-block launch enqueues) for the roofline line."""
    import torch
    from paper_1701_03512_b200 import dist as bpd
    from paper_1701_03512_b200.exact import tree_of
    from paper_1701_03512_b200.payoffs import kind_bit
    req, kinds, P = make_req(w, classic_crr)
    tree, keep = tree_of(req)
    mask = 0
    for k in kinds:
        mask |= 1 << kind_bit(k)
    sh = bpd.ShardedExact(tree, keep, mask, 0, 1, dev)
    st = torch.cuda.current_stream(dev)
    sh.enqueue(st)
    torch.cuda.synchronize(dev)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sh.enqueue(st)
        e1.record(st)
        torch.cuda.synchronize(dev)
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def secondary_configs(dev):
    """BASELINE configs[3] (stratified MC, N=64, k=12, R_m=65536, vs basic MC
    with the same total draws) and configs[4] (4096 Asian calls at N=24)."""
    from types import SimpleNamespace
    import numpy as np
    import paper_1701_03512_b200 as bp
    from paper_1701_03512_b200 import mc as bmc
    out = {}
    N, k, R_m = 64, 12, 65536
    P = bp.classic_crr(N, 0.2, 0.05, 1.0)
    req = object.__new__(bp.ValuationRequest)
    for f, v in dict(inputs=SimpleNamespace(S0=100.0, K=100.0, q=0.05, sigma=0.2, T=1.0, N=N), params=P,
                     kind=bp.ASIAN_CALL, workers=1, force_large=True, devices=[dev]).items():
        object.__setattr__(req, f, v)
    ms = []
    for i in range(4):
        _, _, t = bmc._strata_stats(req, k, [R_m] * (1 << k), 0, 0, 1)
        ms.append(t)
    t = min(ms[1:])
    e = bp.estimate_partitioned_equal(req, bp.McConfig(R=R_m, M=1 << k, seed=0))
    b = bp.estimate_basic(req, bp.McConfig(R=R_m << k, seed=0))
    out["config4"] = {"workload": "stratified MC N=64, k=12 (4096 strata), R_m=65536, Asian call, Philox4x32-10",
                      "value": (R_m << k) / (t * 1e-3), "unit": "draws/s", "kernel_ms": t,
                      "estimate": e.value, "std_error": e.std_error, "basic_estimate": b.value,
                      "basic_std_error": b.std_error, "variance_ratio_basic_over_equal": b.variance / e.variance,
                      "reference_ratio_N62": 1.60, "gpus": 1}
    n, Nb = 4096, 24
    rng = np.random.default_rng(0)
    S0 = rng.uniform(50, 150, n); m = rng.uniform(0.8, 1.2, n); K = m * S0
    sigma = rng.uniform(0.1, 0.5, n); r = rng.uniform(0.0, 0.08, n); T = rng.uniform(0.25, 3.0, n)
    u = np.array([math.exp(a * math.sqrt(b / Nb)) for a, b in zip(sigma, T)])
    d = 1.0 / u
    p = np.array([(math.exp(a * b / Nb) - dd) / (uu - dd) for a, b, uu, dd in zip(r, T, u, d)])
    disc = np.array([math.exp(-a * b) for a, b in zip(r, T)])
    ms = []
    for i in range(3):
        vals, t = bp.price_batch(Nb, S0, K, u, d, p, disc, bp.ASIAN_CALL, device=dev, with_time=True)
        ms.append(t)
    t = min(ms[1:])
    out["config5"] = {"workload": "4096 Asian calls, N=24, parameters from default_rng(0)",
                      "value": n * (1 << Nb) / (t * 1e-3), "unit": "paths/s", "kernel_ms": t,
                      "value_option0": float(vals[0]), "gpus": 1}
    # K8 threshold-search engine: same exact values, leaves counted by binary
    # search (not visited) -> EFFECTIVE paths/s, a separate metric
    wl, classic_crr = workloads()
    srch = {}
    for name in ("config2", "config3"):
        w = wl[name]
        req, kinds, _ = make_req(w, classic_crr)
        ms = []
        for i in range(4):
            r = bp.value_exact(req, kinds=kinds, devices=[dev], search=True)
            ms.append(r.kernel_ms)
        t = min(ms[1:])
        srch[name] = {"effective_paths_per_s": (1 << w["N"]) / (t * 1e-3), "kernel_ms": t, "values": r.values}
    out["threshold_search_engine"] = {"note": "effective paths/s: leaves are counted by binary search over "
                                      "class-sorted tables, not evaluated one by one; not the headline metric",
                                      **srch}
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world
    dev = local
    torch.cuda.set_device(dev)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
    import __graft_entry__
    __graft_entry__.build()
    import paper_1701_03512_b200 as bp
    from paper_1701_03512_b200 import _native

    wl, classic_crr = workloads()
    w = wl[args.workload]
    warmup = max(3, args.warmup)

    with ClockSampler(dev) as clk:
        times, vals, sh, req, kinds = time_workload(w, classic_crr, args.steps, warmup, rank, world, dev, group)
    ms_local = sum(times) / len(times)
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_paths = 1 << w["N"]
    value = total_paths / (ms * 1e-3)

    # config 3 (N = 36) in the same run
    extra = {}
    if args.workload == "config2" and not args.no_config3:
        t3, v3, _, _, _ = time_workload(wl["config3"], classic_crr, max(2, args.steps // 4), 3, rank, world, dev,
                                        group)
        ms3 = sum(t3) / len(t3)
        if world > 1:
            t = torch.tensor([ms3], dtype=torch.float64, device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms3 = float(t.item())
        extra = {"value": (1 << 36) / (ms3 * 1e-3), "unit": "paths/s", "ms_per_step": ms3,
                 "asian_call": v3["asian-call"]}

    # configs[3] (stratified MC, N = 64) and configs[4] (batched exact) on rank 0's GPU
    extra45 = {}
    if rank == 0 and not args.no_config3:
        try:  # secondary numbers must not cost the headline line
            extra45 = secondary_configs(dev)
        except Exception as exc:  # noqa: BLE001
            extra45 = {"secondary_configs_error": f"{type(exc).__name__}: {exc}"}

    # e2e: the public API with host inputs and the result read back every step;
    # for N > 1 every rank takes part (value_exact_distributed: its shard + NCCL)
    e2e_s, e2e_path = e2e_seconds(bp, req, kinds, args, warmup, rank, world, dev, group)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # roofline: FP64-pipe ops (W per path per payoff) / kernel time vs measured DFMA peak
    peak = __import__("ctypes").c_double()
    clk_mhz = __import__("ctypes").c_double()
    _native.check(_native.lib().bp_fp64_peak(dev, __import__("ctypes").byref(peak),
                                             __import__("ctypes").byref(clk_mhz)))
    # the timed steps themselves (CUDA events on the launch stream): at N = 1 a
    # step is K1 + K2 (K1 ~97 % of it, profiles/r1_launches_config2.csv), so
    # this is a slightly conservative K1 duration; the best isolated K1 + K2
    # launch is reported beside it
    k_min_ms = kernel_share(w, classic_crr, dev)
    k_ms = ms_local if world == 1 else k_min_ms  # N > 1: the timed step also holds the NCCL exchange
    W = sum(W_OPS[k] for k in w["kinds"])
    achieved = total_paths * W / (k_ms * 1e-3)
    traffic, ncu = None, None
    try:  # DRAM bytes per launch and pipe counters from the committed ncu --set full capture
        tr = json.load(open(os.path.join(ROOT, "profiles", "r1_traffic.json")))[args.workload]
        traffic = tr["dram_bytes_read"] + tr["dram_bytes_write"]
        ncu = {k: tr[k] for k in ("fp64_pipe_active_pct", "issue_active_pct", "warp_inst_per_32_leaf_tests")}
        ncu["note"] = ("W counts 3 FP64 ops per leaf and payoff; K1 spends ~1.3 (one DSETP + amortised group "
                       "adds), so frac > 1 while the FP64 pipe is ~70 % busy and issue ~90 %")
    except Exception:
        pass
    roof = {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak.value / 1e12, "unit": "Tops/s (FP64 pipe)",
            "frac": achieved / peak.value, "traffic": traffic, "traffic_unit": "bytes/launch (ncu, DRAM)",
            "kernel_ms": k_ms, "kernel_ms_source": "mean of the timed steps (K1 + K2, CUDA events)" if world == 1 else
            "full valuation on one GPU, best of 5 (K1 + K2, CUDA events)",
            "isolated_launch_min_ms": k_min_ms, "W_ops_per_path": W,
            "peak_kind": "measured DFMA microbenchmark (bp_fp64_peak, K7) on this GPU", "ncu": ncu,
            "nominal_peak_Tops": 148 * 64 * 1.965e9 / 1e12}

    h2d = 8 * w["N"] + 7 * 8 + 4  # the tree + per-step probabilities handed to the C ABI
    e2e = {"value": total_paths / e2e_s, "unit": "paths/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": 8 * 6 * 2 * sh.n_sb, "seconds_per_step": e2e_s,
           "path": e2e_path}

    try:
        cpu = cpu_baseline(w, classic_crr) if world == 1 else None
    except Exception as exc:  # noqa: BLE001
        cpu = {"error": f"{type(exc).__name__}: {exc}"}
    launches_per_step = 2 * (1 if set(w["kinds"]) == {"asian-call", "float-lookback"} else len(w["kinds"]))
    line = {
        "metric": METRIC,
        "value": value, "unit": "paths/s", "n_gpus": world, "steps": args.steps, "warmup": warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE configs; tree parameters, no dataset)",
        "config": {**workload_config(args.workload, w), "parallelism": f"superblock-shard x{world}",
                   "l2": "flushed (256 MiB write) between timed steps", "engine": "affine-threshold" if sh.engine else
                   "path-walk", "inner_bits": sh.inner_bits, "superblocks": sh.n_sb},
        "values": vals, "config3": extra or None, **extra45, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config2", choices=["config1", "config2", "config3"])
    ap.add_argument("--no-config3", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
