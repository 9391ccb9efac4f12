"""Benchmark: exact-enumeration paths/s on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload config2|config3|config1]

One step = one exact valuation of the workload's tree: every one of the 2^N
paths evaluated (both payoffs of config 2 in one pass), the per-rank
super-block partials reduced, exchanged (NCCL all_gather when N > 1) and
combined.  Default workload = BASELINE configs[1] (N = 30, Asian call +
floating lookback, K from default_rng(0)); config 3 (N = 36 Asian call) is
measured in the same run and reported under "config3".

--gpus N > 1 re-executes itself under torchrun with N ranks, one per GPU
(paper_1701_03512_b200.launch); fewer than N visible GPUs is an error, never
a silent one-GPU run.  Each rank owns a contiguous range of the 64 canonical
super-blocks; the total 2^N work is fixed, so "scaling" is "strong".

--impl reference times the reference algorithm on the host CPU: the C
restatement in oracle/ (the reference is pure Python and cannot be compiled)
on every host thread, whole valuations per step when they fit the run's
time budget.  The stock reference package (baseline/_ref, numpy) is timed
beside it at N = 24 as a labelled second baseline.
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
FP64_LANES_PER_SM = 64   # B200: 64 FP64 lanes per SM per clock
FP32_LANES_PER_SM = 128
REF_BUDGET_S = 240.0     # the reference arm's whole run (all steps) stays within this


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
    """The workload keys both arms report (identical config for the driver's ratio)."""
    return {"workload": name, "N": w["N"], "payoffs": w["kinds"], "K": w["K"], "S0": w["S0"], "r": w["r"],
            "sigma": w["sigma"], "T": w["T"]}


def make_req(w, classic_crr):
    import paper_1701_03512_b200 as bp
    P = classic_crr(w["N"], w["sigma"], w["r"], w["T"])
    inputs = bp.MarketInputs(S0=w["S0"], K=w["K"], q=w["r"], sigma=w["sigma"], T=w["T"], N=w["N"])
    kinds = [bp.resolve_kind(k) for k in w["kinds"]]
    return bp.ValuationRequest(inputs=inputs, params=P, kind=kinds[0], force_large=True), kinds, P


def load_counters(workload):
    """Per-launch counters of the dominant kernel from the committed ncu
    capture of this instantiation (profiles/r2_kernel_counters.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_kernel_counters.json")) as f:
            return json.load(f)[workload]
    except Exception:  # noqa: BLE001
        return None


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
# CPU baselines (the only place bench.py runs oracle/ or the stock reference)
def _oracle_paths(w, classic_crr, n, threads):
    import oracle
    P = classic_crr(w["N"], w["sigma"], w["r"], w["T"])
    disc = math.exp(-w["r"] * w["T"])
    t0 = time.perf_counter()
    vals, paths = oracle.exact_range(w["N"], w["S0"], w["K"], P.u, P.d, P.up_probs[0], disc, w["kinds"], 0, n,
                                     threads)
    return paths, time.perf_counter() - t0, vals


def cpu_baseline(w, classic_crr, budget_s=12.0):
    """Reference algorithm (oracle/ C restatement) on every host thread, on a
    bounded contiguous sample of the workload's path codes."""
    threads = os.cpu_count() or 1
    n = 1 << 16
    while True:
        paths, elapsed, _ = _oracle_paths(w, classic_crr, n, threads)
        if elapsed * 4 > budget_s or n >= (1 << w["N"]):
            break
        n <<= 2
    return {"value": paths / elapsed, "unit": "paths/s", "cores": threads, "kind": "port",
            "sample": f"{paths} of 2^{w['N']} paths (codes [0, {paths})), {'+'.join(w['kinds'])} in one pass, "
                      f"{elapsed:.2f} s wall, oracle/bp_oracle.c (per-path walk as exact.py:83-100)"}


def stock_reference_baseline(N=24):
    """The UNMODIFIED reference package (baseline/_ref, numpy) on this host:
    value_exact_parallel(workers=os.cpu_count()) on config 2's lattice at
    N = 24.  It has no Asian call / floating lookback
    built-in: Asian call = ASIAN_PUT at (-S0, -K) (bit-identical to the
    callable route), floating lookback = FIXED_LOOKBACK_PUT(-S0, 0) -
    EUROPEAN_CALL(S0, 0); the three engine walls are summed."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "binpaths")):
        return {"unavailable": "baseline/_ref not installed (see DESIGN.md)"}
    sys.path.insert(0, ref)
    try:
        from types import SimpleNamespace

        import numpy as np
        import binpaths as B
        wl, _ = workloads()
        w = wl["config2"]
        S0, K, r, sigma, T = w["S0"], w["K"], w["r"], w["sigma"], w["T"]
        dt = T / N
        u = math.exp(sigma * math.sqrt(dt))
        d = 1 / u
        p = (math.exp(r * dt) - d) / (u - d)
        P = B.TreeParams(dt=dt, u=u, d=d, beta=0.5 * (u + d), up_probs=np.full(N, p))
        cores = os.cpu_count() or 1

        def run(kind, s0, k):
            req = B.ValuationRequest(inputs=SimpleNamespace(S0=s0, K=k, q=r, T=T, N=N), params=P, kind=kind,
                                     workers=cores, force_large=True)
            t0 = time.perf_counter()
            v = B.value_exact_parallel(req)
            return v, time.perf_counter() - t0

        ac, t1 = run(B.PayoffKind.ASIAN_PUT, -S0, -K)
        flp, t2 = run(B.PayoffKind.FIXED_LOOKBACK_PUT, -S0, 0.0)
        ec, t3 = run(B.PayoffKind.EUROPEAN_CALL, S0, 0.0)
        wall = t1 + t2 + t3
        return {"value": (1 << N) / wall, "unit": "paths/s", "cores": cores, "kind": "reference",
                "sample": f"stock binpaths {getattr(B, '__version__', '0.1.0')} (baseline/_ref), "
                          f"value_exact_parallel(workers={cores}), config-2 lattice at N={N}: Asian call by the "
                          f"sign-flip route + floating lookback as two runs, 3 engine walls summed = {wall:.2f} s",
                "values": {"asian-call": ac, "float-lookback": flp - ec}}
    except Exception as exc:  # noqa: BLE001
        return {"unavailable": f"{type(exc).__name__}: {exc}"}
    finally:
        sys.path.remove(ref)


def run_reference(args):
    """The reference arm: rank 0 only (other torchrun ranks exit 0)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    wl, classic_crr = workloads()
    w = wl[args.workload]
    threads = os.cpu_count() or 1
    full = 1 << w["N"]
    # size each step so the whole run stays within the budget: whole
    # valuations when they fit, else the largest power-of-two code prefix
    cal_n = min(full, 1 << 22)
    _, cal_t, _ = _oracle_paths(w, classic_crr, cal_n, threads)
    per_path = cal_t / cal_n
    n = full
    while n > cal_n and per_path * n * (args.steps + args.warmup) > REF_BUDGET_S:
        n >>= 1
    ts, paths = [], 0
    for i in range(args.warmup + args.steps):
        p, t, vals = _oracle_paths(w, classic_crr, n, threads)
        if i >= args.warmup:
            ts.append(t)
            paths = p
    sec = sum(ts) / len(ts)
    v = paths / sec
    sample = (f"{'whole valuation' if n == full else 'code prefix'}: {paths} of 2^{w['N']} paths per step "
              f"(codes [0, {paths})), {'+'.join(w['kinds'])} in one pass, {sec:.2f} s per step, "
              f"oracle/bp_oracle.c (per-path walk as exact.py:83-100) on {threads} threads")
    line = {"metric": METRIC, "value": v, "unit": "paths/s",
            "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE configs; tree parameters, no dataset)", "impl": "reference",
            "config": workload_config(args.workload, w),
            "impl_detail": {"parallelism": f"{threads} host threads", "whole_valuation_per_step": n == full},
            "cpu_baseline": {"value": v, "unit": "paths/s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if n == full:
        line["values"] = vals
    if not args.no_stock:
        line["stock_reference"] = stock_reference_baseline()
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def time_workload(w, classic_crr, steps, warmup, rank, world, dev, group):
    """Device-timed steps (CUDA events on the launch stream), L2 flushed
    between steps.  A step = this rank's super-blocks (K1 + K2) and, for
    N > 1, the all_gather.  Also times the two halves alone: the rank's
    kernels (its roofline) and the exchange (the fixed multi-GPU cost)."""
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

    def timed(fn, n):
        out = []
        for _ in range(n):
            flush.fill_(1)
            if world > 1:
                dist.barrier(group=group)
            torch.cuda.synchronize(dev)
            e0, e1 = _events(torch)
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize(dev)
            out.append(e0.elapsed_time(e1))
        return out

    def step():
        sh.enqueue(st)
        sh.exchange(group)

    times = timed(step, steps)
    vals = sh.values()
    detail = {}
    kern = timed(lambda: sh.enqueue(st), max(3, min(steps, 10)))
    detail["kernel_ms"] = sum(kern) / len(kern)
    if world > 1:
        xch = timed(lambda: sh.exchange(group), max(3, min(steps, 10)))
        detail["exchange_ms"] = sum(xch) / len(xch)
    detail["superblocks"] = (sh.first, sh.count, sh.n_sb)
    return times, vals, sh, req, kinds, detail


def _max_over_ranks(x, world, dev):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _gather_ranks(x, world, dev):
    if world == 1:
        return [x]
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}")
    out = torch.empty(world, dtype=torch.float64, device=f"cuda:{dev}")
    dist.all_gather_into_tensor(out, t)
    return [float(v) for v in out.cpu()]


def e2e_seconds(bp, req, kinds, args, warmup, rank, world, dev, group):
    """Median wall seconds of one public-API valuation (host request in,
    Python floats out), max over ranks.  N = 1: value_exact (C ABI, one
    synchronous call); N > 1: value_exact_distributed on every rank (this
    rank's super-blocks, the NCCL all_gather, the host combine)."""
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
    med = _max_over_ranks(statistics.median(ts), world, dev)
    if world > 1:
        return med, "paper_1701_03512_b200.dist.value_exact_distributed(req, kinds, rank, world) on every rank"
    return med, "paper_1701_03512_b200.value_exact(req, kinds) -> bp_exact (C ABI)"


def fp64_peak(dev):
    """K7: the measured DFMA rate and the SM clock K7 ran at."""
    import ctypes
    from paper_1701_03512_b200 import _native
    rate, mhz = ctypes.c_double(), ctypes.c_double()
    _native.check(_native.lib().bp_fp64_peak(dev, ctypes.byref(rate), ctypes.byref(mhz)))
    return rate.value, mhz.value


# Leaf-test forms of K1 and their peak rates per SM sub-partition per clock,
# measured on this B200 (tools/microbench, profiles/r2_microbench_*.log):
# any SETP (DSETP included) issues at 0.5 warp-instructions/clk -> 16 leaf
# tests; the I15 screen's packed IMAD (two nodes' 15-bit lanes per 32-bit
# lane) at 0.5 warp-instructions/clk -> 32 leaf tests.
TESTS_PER_CLK_SMSP = {"fp64": 16.0, "i15": 32.0}


def i15_share(L):
    """Share of an inner block's 2^L leaves in up-count classes with >= 16
    leaves (the screened ones; csrc/bp_exact.cuh i15_class)."""
    return sum(math.comb(L, c) for c in range(L + 1) if math.comb(L, c) >= 16) / float(1 << L)


def leaf_test_mix(kinds, L):
    """(form, tests per path) of K1's leaf tests for the workload's kinds:
    every table kind (Asian and lookback) screens its big up-count classes
    (I15) and tests the small classes in fp64 (csrc/bp_exact_fast.cuh)."""
    mix = {"fp64": 0.0, "i15": 0.0}
    for _ in kinds:
        mix["i15"] += i15_share(L)
        mix["fp64"] += 1.0 - i15_share(L)
    return mix


def roofline(w, workload, k_ms, paths, sm_count, clk, dev, inner_bits=9):
    """Compare roofline of the dominant kernel (K1, with K2 inside k_ms).

    The algorithmic unit is the leaf test (one explicit compare per leaf per
    payoff).  peak = the leaf-test rate of K1's own compare forms at their
    measured pipe peak (TESTS_PER_CLK_SMSP), mixed in this workload's
    proportions, x 4 sub-partitions x n_SM x the SM clock sampled during the
    timed region; achieved = leaf tests per launch / kernel time; frac =
    achieved / peak <= 1.  The ncu counters of the committed capture of this
    instantiation (issue utilisation, warp instructions per leaf test, FP64
    pipe) say where the rest of the time goes.  fp64_context keeps the
    SURVEY §8d FP64-pipe figures: the W-based fraction (3 FP64 ops per path
    per payoff, > 1 because K1 tests most leaves off the FP64 pipe) and the
    K7 DFMA microbenchmark."""
    k7_rate, k7_mhz = fp64_peak(dev)
    mhz = (clk or {}).get("sm_mhz") or k7_mhz
    hz = mhz * 1e6
    tests = paths * len(w["kinds"])
    mix = leaf_test_mix(w["kinds"], inner_bits)
    # seconds per path at the compare peak, per form
    sec_per_path = sum(share / (TESTS_PER_CLK_SMSP[f] * 4 * sm_count * hz) for f, share in mix.items())
    peak = len(w["kinds"]) / sec_per_path  # leaf tests / s
    achieved = tests / (k_ms * 1e-3)
    roof = {"bound": "compare", "unit": "leaf tests/s (x1e12)", "achieved": achieved / 1e12, "peak": peak / 1e12,
            "frac": achieved / peak,
            "peak_kind": (f"K1 leaf-test forms at their measured pipe peaks ({', '.join(f'{k} {v:g}' for k, v in TESTS_PER_CLK_SMSP.items())} "
                          f"tests/clk/SMSP, profiles/r2_microbench_*.log) in this workload's mix "
                          f"({', '.join(f'{k} {v:.3f}' for k, v in mix.items())} tests per path) x 4 x {sm_count} SMs "
                          f"x {mhz:.0f} MHz (SM clock sampled during the timed region)"),
            "kernel_ms": k_ms, "paths_per_launch": paths, "leaf_tests_per_launch": tests}
    c = load_counters(workload)
    if c:
        roof.update({"traffic": c["dram_bytes_read"] + c["dram_bytes_write"],
                     "traffic_unit": "DRAM bytes per launch (ncu)",
                     "ncu": {k: c[k] for k in ("issue_active_pct", "warp_inst_per_32_leaf_tests",
                                               "fp64_pipe_active_pct", "alu_pipe_active_pct", "fma_pipe_active_pct",
                                               "fp64_pipe_ops_per_leaf_test", "source")
                             if k in c}})
    else:
        roof.update({"traffic": None})
    fp64_peak_ops = sm_count * FP64_LANES_PER_SM * hz
    W = sum(W_OPS[k] for k in w["kinds"])
    roof["fp64_context"] = {
        "peak_tops": fp64_peak_ops / 1e12,
        "frac_w": paths * W / (k_ms * 1e-3) / fp64_peak_ops, "W_ops_per_path": W,
        "note": "SURVEY 8d W-based FP64 figure: 3 FP64 ops per path per payoff over the FP64-pipe peak "
                f"({sm_count} SMs x {FP64_LANES_PER_SM} lanes x {mhz:.0f} MHz); above 1 because K1 screens most "
                "leaves with 15-bit integer compares and spends FP64 only on the lookback leaves, the small "
                "classes and the ambiguous boundary leaf",
        "k7": {"dfma_per_s": k7_rate, "sm_mhz": k7_mhz,
               "frac_of_pipe_at_its_clock": k7_rate / (sm_count * FP64_LANES_PER_SM * k7_mhz * 1e6)
               if k7_mhz else None}}
    roof["fp32_context"] = {"peak_tflops": 2 * FP32_LANES_PER_SM * sm_count * hz / 1e12,
                            "note": "FMA-pipe peak at the same clock (FMA = 2 flops); the screen's packed IMAD runs "
                                    "on the FMA pipe (ncu fma_pipe_active_pct)"}
    return roof


def secondary_configs(dev):
    """BASELINE configs[3] (stratified MC, N=64, k=12, R_m=65536, vs basic MC
    with the same total draws) and configs[4] (4096 Asian calls at N=24)."""
    from types import SimpleNamespace
    import numpy as np
    import paper_1701_03512_b200 as bp
    from paper_1701_03512_b200 import mc as bmc
    out = {}
    # configs[0] (N = 20, the reference's own CPU-runnable case): launch-bound on a GPU
    wl1, crr1 = workloads()
    req1, kinds1, _ = make_req(wl1["config1"], crr1)
    r1 = [bp.value_exact(req1, kinds=kinds1, devices=[dev]) for _ in range(8)]
    t0 = time.perf_counter()
    for _ in range(50):
        bp.value_exact(req1, kinds=kinds1, devices=[dev])
    call_s = (time.perf_counter() - t0) / 50
    k1 = min(r.kernel_ms for r in r1[2:])
    out["config1"] = {"workload": "exact Asian call, N=20 (2^20 paths): launch-bound on a GPU",
                      "kernel_ms": k1, "call_ms": call_s * 1e3, "value": (1 << 20) / call_s, "unit": "paths/s",
                      "asian_call": r1[-1].values["asian-call"]}
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
    t0 = time.perf_counter()
    e = bp.estimate_partitioned_equal(req, bp.McConfig(R=R_m, M=1 << k, seed=0))
    call4_ms = (time.perf_counter() - t0) * 1e3  # the public estimator call: host in, Estimate out
    b = bp.estimate_basic(req, bp.McConfig(R=R_m << k, seed=0))
    out["config4"] = {"workload": "stratified MC N=64, k=12 (4096 strata), R_m=65536, Asian call, Philox4x32-10",
                      "value": (R_m << k) / (t * 1e-3), "unit": "draws/s", "kernel_ms": t, "call_ms": call4_ms,
                      "estimate": e.value, "std_error": e.std_error, "basic_estimate": b.value,
                      "basic_std_error": b.std_error, "variance_ratio_basic_over_equal": b.variance / e.variance,
                      "reference_ratio_N62": 1.60, "gpus": 1,
                      "sampler": {"philox_blocks_per_draw": 4.5,
                                  "philox_blocks_per_s": 4.5 * (R_m << k) / (t * 1e-3),
                                  "philox_ceiling_blocks_per_s": 5.15e11,
                                  "frac_of_philox_ceiling": 4.5 * (R_m << k) / (t * 1e-3) / 5.15e11,
                                  "warp_inst_per_draw": 353.4,
                                  "note": "bit-sliced sampler: 8 threshold bits decided 32 steps per Philox word, "
                                          "tie words for the 2^-8 rest (exactly floor(p 2^32)/2^32 per step); "
                                          "ceiling = Philox4x32-10 alone, tools/microbench/mb_philox.cu "
                                          "(profiles/r1_microbench_philox.log); instruction count from "
                                          "profiles/r2_config4_full.ncu-rep"}}
    n, Nb = 4096, 24
    rng = np.random.default_rng(0)
    S0 = rng.uniform(50, 150, n); m = rng.uniform(0.8, 1.2, n); K = m * S0
    sigma = rng.uniform(0.1, 0.5, n); r = rng.uniform(0.0, 0.08, n); T = rng.uniform(0.25, 3.0, n)
    u = np.array([math.exp(a * math.sqrt(b / Nb)) for a, b in zip(sigma, T)])
    d = 1.0 / u
    p = np.array([(math.exp(a * b / Nb) - dd) / (uu - dd) for a, b, uu, dd in zip(r, T, u, d)])
    disc = np.array([math.exp(-a * b) for a, b in zip(r, T)])
    ms, calls = [], []
    for i in range(3):
        t0 = time.perf_counter()
        vals, t = bp.price_batch(Nb, S0, K, u, d, p, disc, bp.ASIAN_CALL, device=dev, with_time=True)
        calls.append((time.perf_counter() - t0) * 1e3)
        ms.append(t)
    t = min(ms[1:])
    out["config5"] = {"workload": "4096 Asian calls, N=24, parameters from default_rng(0)",
                      "value": n * (1 << Nb) / (t * 1e-3), "unit": "paths/s", "kernel_ms": t,
                      "call_ms": min(calls[1:]), "value_option0": float(vals[0]), "gpus": 1}
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
    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    group = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
    import __graft_entry__
    __graft_entry__.build()
    import paper_1701_03512_b200 as bp

    wl, classic_crr = workloads()
    w = wl[args.workload]
    warmup = max(3, args.warmup)

    with ClockSampler(dev) as clk:
        times, vals, sh, req, kinds, detail = time_workload(w, classic_crr, args.steps, warmup, rank, world, dev,
                                                            group)
    ms_local = sum(times) / len(times)
    ms = _max_over_ranks(ms_local, world, dev)
    total_paths = 1 << w["N"]
    value = total_paths / (ms * 1e-3)
    clocks = clk.summary()

    # config 3 (N = 36) in the same run
    extra = {}
    if args.workload == "config2" and not args.no_config3:
        t3, v3, _, _, _, _ = time_workload(wl["config3"], classic_crr, max(2, args.steps // 4), 3, rank, world,
                                           dev, group)
        ms3 = _max_over_ranks(sum(t3) / len(t3), world, dev)
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

    per_rank_ms = _gather_ranks(ms_local, world, dev)
    per_rank_kernel_ms = _gather_ranks(detail["kernel_ms"], world, dev)
    per_rank_exchange_ms = _gather_ranks(detail.get("exchange_ms", 0.0), world, dev)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    # roofline of the dominant kernel on this rank: its share of the super-blocks
    first, count, n_sb = detail["superblocks"]
    rank_paths = total_paths * count // n_sb
    k_ms = ms_local if world == 1 else detail["kernel_ms"]
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    roof = roofline(w, args.workload, k_ms, rank_paths, sm_count, clocks, dev, sh.inner_bits)
    roof["kernel_ms_source"] = ("mean of the timed steps (K1 + K2, CUDA events on the launch stream)" if world == 1
                                else "rank 0's super-blocks alone (K1 + K2, CUDA events), no exchange")

    h2d = 8 * w["N"] + 7 * 8 + 4  # the tree + per-step probabilities handed to the C ABI
    e2e = {"value": total_paths / e2e_s, "unit": "paths/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": 8 * 6 * 2 * sh.n_sb, "seconds_per_step": e2e_s, "path": e2e_path}

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
        "config": workload_config(args.workload, w),
        "impl_detail": {"parallelism": f"superblock-shard x{world} (one rank per GPU, NCCL all_gather)",
                        "l2": "flushed (256 MiB write) between timed steps",
                        "engine": "affine-threshold" if sh.engine else "path-walk", "inner_bits": sh.inner_bits,
                        "superblocks": sh.n_sb, "leaf_block": "15-bit integer screen of the big up-count "
                                                             "classes (two nodes per IMAD, Gray-code counters, fp64 "
                                                             "boundary leaf); small classes: fp64 compares with "
                                                             "Gray-code predicate counting; per-class fold, 2 nodes "
                                                             "per table load"},
        "values": vals, "config3": extra or None, **extra45, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
    }
    if world > 1:
        line["scaling_detail"] = {"per_rank_step_ms": per_rank_ms, "per_rank_kernel_ms": per_rank_kernel_ms,
                                  "per_rank_exchange_ms": per_rank_exchange_ms,
                                  "note": "step = the rank's K1 + K2 and the NCCL all_gather; kernel / exchange "
                                          "timed alone with CUDA events (means), max over ranks for the step"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config2", choices=["config1", "config2", "config3"])
    ap.add_argument("--no-config3", action="store_true", help="headline workload only (no secondary configs)")
    ap.add_argument("--no-stock", action="store_true", help="reference arm: skip the stock-package baseline")
    args = ap.parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    from paper_1701_03512_b200.launch import LaunchError, ensure_world
    try:
        rc = ensure_world(args.gpus, __file__, argv)
    except LaunchError as exc:
        print(f"bench.py: {exc}", file=sys.stderr)
        return 2
    if rc is not None:  # ran the ranks under torchrun
        return rc
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
