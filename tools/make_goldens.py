"""Generate golden vectors from the reference `binpaths` package.

This script imports the UNMODIFIED reference from /root/reference/pkg/src
(present only in the build container; it does not travel to the GPU box)
and writes small JSON fixtures under tests/golden/.  The fixtures pin the
CPU oracle (oracle/) and, through it, the CUDA path.

Routes used for the two BASELINE payoffs the reference has no enum tag for
(SURVEY.md §8c):
  * Asian call       = ASIAN_PUT evaluated with (S0, K) -> (-S0, -K)
  * floating lookback = FIXED_LOOKBACK_PUT(-S0, K=0) - EUROPEAN_CALL(S0, K=0)
For small N the reference's own callable extension point
(payoffs.py:66-70, 94-101) is used as well, so the routes are cross-checked.

Usage:
  python tools/make_goldens.py small            # seconds
  python tools/make_goldens.py config1          # ~10 s
  python tools/make_goldens.py config2          # ~5 min on 8 cores
  python tools/make_goldens.py paper            # ~10 min on 8 cores
  python tools/make_goldens.py batch            # ~30 s on 8 cores
  python tools/make_goldens.py mc               # ~2 min
  python tools/make_goldens.py config3          # ~90 min on 8 cores
  python tools/make_goldens.py cli              # seconds
"""

from __future__ import annotations

import json
import math
import os
import platform
import sys
import time
from types import SimpleNamespace

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import binpaths as bp  # noqa: E402  (the reference package)
from binpaths import (  # noqa: E402
    McConfig,
    MarketInputs,
    PayoffKind,
    TreeParams,
    ValuationRequest,
    allocate_strata,
    asset_path,
    block_probability,
    derive_crr,
    estimate_basic,
    estimate_partitioned,
    estimate_partitioned_equal,
    estimate_shared,
    make_partition,
    run_repetitions,
    value_exact_parallel,
    value_exact_serial,
    with_custom_probs,
)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
CORES = os.cpu_count() or 1


def provenance(extra=None):
    d = {
        "generator": "tools/make_goldens.py",
        "reference": "binpaths " + getattr(bp, "__version__", "?") + " from /root/reference/pkg/src",
        "numpy": np.__version__,
        "python": platform.python_version(),
        "cores": CORES,
    }
    if extra:
        d.update(extra)
    return d


def dump(name, payload):
    path = os.path.join(OUT, name)
    with open(path, "w") as f:
        json.dump(payload, f, indent=1, sort_keys=False)
    print("wrote", path)


def classic_crr(N, sigma, r, T):
    """BASELINE.json lattice: u=exp(sigma sqrt dt), d=1/u, p=(e^{r dt}-d)/(u-d)."""
    dt = T / N
    u = math.exp(sigma * math.sqrt(dt))
    d = 1.0 / u
    p = (math.exp(r * dt) - d) / (u - d)
    return TreeParams(dt=dt, u=u, d=d, beta=0.5 * (u + d), up_probs=np.full(N, p))


def value(kind, params, S0, K, q, T, N, workers=1, serial=False):
    inputs = SimpleNamespace(S0=S0, K=K, q=q, T=T, N=N)
    req = ValuationRequest(inputs=inputs, params=params, kind=kind,
                           workers=workers, force_large=True)
    return value_exact_serial(req) if serial else value_exact_parallel(req)


def asian_call_route(params, S0, K, q, T, N, workers=1, serial=False):
    return value(PayoffKind.ASIAN_PUT, params, -S0, -K, q, T, N, workers, serial)


def float_lookback_route(params, S0, q, T, N, workers=1, serial=False):
    a = value(PayoffKind.FIXED_LOOKBACK_PUT, params, -S0, 0.0, q, T, N, workers, serial)
    b = value(PayoffKind.EUROPEAN_CALL, params, S0, 0.0, q, T, N, workers, serial)
    return a - b, a, b


# callables through the reference's extension point (payoffs.py:66-70)
def cb_asian_call(params, S0, K, path):
    return float(max(asset_path(params, S0, path).mean() - K, 0.0))


def cb_float_lookback(params, S0, K, path):
    s = asset_path(params, S0, path)
    return float(s.max() - s[-1])


def params_record(params):
    return {"u": params.u, "d": params.d, "up_probs": [float(x) for x in params.up_probs]}


# --------------------------------------------------------------------------
def gen_small():
    """All kinds, N=1..12, random lattices incl. per-step probabilities."""
    rng = np.random.default_rng(20260101)
    cases = []
    builtin = [PayoffKind.EUROPEAN_CALL, PayoffKind.EUROPEAN_PUT,
               PayoffKind.ASIAN_PUT, PayoffKind.FIXED_LOOKBACK_PUT]

    def add_case(tag, N, S0, K, q, T, params):
        vals = {}
        for kind in builtin:
            vals[kind.value] = value(kind, params, S0, K, q, T, N, serial=True)
        vals["asian-call"] = value(cb_asian_call, params, S0, K, q, T, N, serial=True)
        vals["float-lookback"] = value(cb_float_lookback, params, S0, K, q, T, N, serial=True)
        route_ac = asian_call_route(params, S0, K, q, T, N, serial=True)
        route_fl = float_lookback_route(params, S0, q, T, N, serial=True)[0]
        cases.append({"tag": tag, "N": N, "S0": S0, "K": K, "q": q, "T": T,
                      **params_record(params), "values": vals,
                      "route_asian_call": route_ac, "route_float_lookback": route_fl})

    # the reference's hand-enumerated toy tree (tests/test_exact.py:28-39)
    toy = TreeParams(dt=0.5, u=2.0, d=0.5, beta=1.25, up_probs=np.full(2, 0.5))
    add_case("toy", 2, 4.0, 5.0, 0.0, 1.0, toy)

    for N in range(1, 13):
        for j in range(2):
            S0 = float(rng.uniform(20, 150))
            K = float(S0 * rng.uniform(0.8, 1.2))
            q = float(rng.uniform(-0.02, 0.1))
            sigma = float(rng.uniform(0.1, 1.0))
            T = float(rng.uniform(0.25, 2.0))
            if j == 0:
                params = classic_crr(N, sigma, max(q, 0.0), T)
            else:
                params = derive_crr(MarketInputs(S0=S0, K=K, q=q, sigma=sigma, T=T, N=N))
            add_case(f"N{N}_{'classic' if j == 0 else 'beta'}", N, S0, K, q, T, params)
    # per-step probabilities (model.py:152-161)
    for N in (3, 7, 11):
        S0, K, q, sigma, T = 50.0, 52.0, 0.03, 0.4, 1.0
        inputs = MarketInputs(S0=S0, K=K, q=q, sigma=sigma, T=T, N=N)
        probs = rng.uniform(0.2, 0.8, size=N)
        params = with_custom_probs(inputs, probs)
        add_case(f"N{N}_custom", N, S0, K, q, T, params)
    # d != 1/u lattice (the engine accepts any TreeParams, exact.py:38-56)
    for N in (5, 10):
        params = TreeParams(dt=1.0 / N, u=1.12, d=0.93, beta=1.0, up_probs=np.full(N, 0.45))
        add_case(f"N{N}_skew", N, 40.0, 41.0, 0.01, 1.0, params)
    # sigma = 0 (p == 1 exactly, model.py:128-132)
    inputs = MarketInputs(S0=2.0, K=1.0, q=0.05, sigma=0.0, T=1.0, N=6)
    add_case("sigma0", 6, 2.0, 1.0, 0.05, 1.0, derive_crr(inputs))

    # medium N (16..20) through the fast routes only
    medium = []
    for N in (13, 14, 16, 18, 20):
        S0 = float(rng.uniform(50, 150)); K = float(S0 * rng.uniform(0.85, 1.15))
        r = float(rng.uniform(0.0, 0.08)); sigma = float(rng.uniform(0.1, 0.5)); T = float(rng.uniform(0.25, 3.0))
        params = classic_crr(N, sigma, r, T)
        vals = {k.value: value(k, params, S0, K, r, T, N, workers=CORES) for k in builtin}
        vals["asian-call"] = asian_call_route(params, S0, K, r, T, N, workers=CORES)
        vals["float-lookback"] = float_lookback_route(params, S0, r, T, N, workers=CORES)[0]
        medium.append({"tag": f"N{N}_medium", "N": N, "S0": S0, "K": K, "q": r, "T": T,
                       "u": params.u, "d": params.d, "p": float(params.up_probs[0]),
                       "values": vals})

    # partition / allocation / block masses (paths.py:103-167, mc.py:162-194)
    parts = []
    for n, m in [(6, 1), (6, 4), (10, 8), (10, 3), (12, 5), (9, 7), (20, 8)]:
        pp = make_partition(n, m)
        parts.append({"n": n, "m": m, "prefix_width": pp.prefix_width,
                      "blocks": [list(b) for b in pp.blocks]})
    allocs = []
    for _ in range(60):
        n = int(rng.integers(3, 13))
        m = 1 << int(rng.integers(0, min(n, 6) + 1))
        R = int(rng.integers(m, 5000))
        probs = rng.uniform(0.05, 0.95, size=n)
        params = TreeParams(dt=1.0, u=1.1, d=1 / 1.1, beta=1.0, up_probs=probs)
        pp = make_partition(n, m)
        allocs.append({"n": n, "m": m, "R": R, "up_probs": [float(x) for x in probs],
                       "alloc": allocate_strata(pp, params, R),
                       "masses": [block_probability(params, pp, k) for k in range(m)]})
    for probs, m, R in [([0.9, 0.5, 0.5, 0.5], 2, 1024), ([0.999, 0.5, 0.5, 0.5], 2, 10),
                        ([0.5] * 6, 4, 1024), ([1.0] * 8, 4, 8)]:
        n = len(probs)
        params = TreeParams(dt=1.0, u=1.1, d=1 / 1.1, beta=1.0, up_probs=np.array(probs))
        pp = make_partition(n, m)
        allocs.append({"n": n, "m": m, "R": R, "up_probs": probs,
                       "alloc": allocate_strata(pp, params, R),
                       "masses": [block_probability(params, pp, k) for k in range(m)]})
    crr = []
    for _ in range(20):
        inputs = MarketInputs(S0=1.0, K=1.0, q=float(rng.uniform(-0.05, 0.2)),
                              sigma=float(rng.uniform(0.01, 2.0)), T=float(rng.uniform(0.1, 3.0)),
                              N=int(rng.integers(1, 63)))
        pr = derive_crr(inputs)
        crr.append({"q": inputs.q, "sigma": inputs.sigma, "T": inputs.T, "N": inputs.N,
                    "dt": pr.dt, "u": pr.u, "d": pr.d, "beta": pr.beta, "p": float(pr.up_probs[0])})
    dump("exact_small.json", {"provenance": provenance(), "cases": cases, "medium": medium,
                              "partitions": parts, "allocations": allocs, "derive_crr": crr})


def gen_config1():
    N, S0, K, r, sigma, T = 20, 100.0, 100.0, 0.05, 0.2, 1.0
    params = classic_crr(N, sigma, r, T)
    t0 = time.time()
    ac = asian_call_route(params, S0, K, r, T, N, workers=CORES)
    fl, fl_max, fl_end = float_lookback_route(params, S0, r, T, N, workers=CORES)
    aput = value(PayoffKind.ASIAN_PUT, params, S0, K, r, T, N, workers=CORES)
    lput = value(PayoffKind.FIXED_LOOKBACK_PUT, params, S0, K, r, T, N, workers=CORES)
    wall = time.time() - t0
    dump("exact_config1.json", {"provenance": provenance({"wall_s": wall}),
                                "config": "BASELINE configs[0]", "N": N, "S0": S0, "K": K, "r": r,
                                "sigma": sigma, "T": T, "u": params.u, "d": params.d,
                                "p": float(params.up_probs[0]),
                                "asian_call": ac, "float_lookback": fl,
                                "float_lookback_parts": [fl_max, fl_end],
                                "asian_put": aput, "fixed_lookback_put": lput})


def gen_config2():
    N, S0, r, sigma, T = 30, 100.0, 0.05, 0.2, 1.0
    K = float(np.random.default_rng(0).uniform(80, 120))
    params = classic_crr(N, sigma, r, T)
    t0 = time.time()
    ac = asian_call_route(params, S0, K, r, T, N, workers=CORES)
    t1 = time.time()
    fl, fl_max, fl_end = float_lookback_route(params, S0, r, T, N, workers=CORES)
    t2 = time.time()
    dump("exact_config2.json", {"provenance": provenance({"wall_s_asian": t1 - t0, "wall_s_lookback": t2 - t1}),
                                "config": "BASELINE configs[1]", "N": N, "S0": S0, "K": K,
                                "K_rule": "numpy.random.default_rng(0).uniform(80,120)",
                                "r": r, "sigma": sigma, "T": T,
                                "u": params.u, "d": params.d, "p": float(params.up_probs[0]),
                                "asian_call": ac, "float_lookback": fl,
                                "float_lookback_parts": [fl_max, fl_end]})


def gen_config3():
    N, S0, K, r, sigma, T = 36, 100.0, 105.0, 0.03, 0.3, 2.0
    params = classic_crr(N, sigma, r, T)
    t0 = time.time()
    ac = asian_call_route(params, S0, K, r, T, N, workers=CORES)
    dump("exact_config3.json", {"provenance": provenance({"wall_s": time.time() - t0}),
                                "config": "BASELINE configs[2]", "N": N, "S0": S0, "K": K,
                                "r": r, "sigma": sigma, "T": T,
                                "u": params.u, "d": params.d, "p": float(params.up_probs[0]),
                                "asian_call": ac})


def gen_paper():
    # beta-CRR lattice through derive_crr, N=32
    inputs = MarketInputs(S0=20.0, K=100.0, q=0.06, sigma=3.0, T=1.0, N=32)
    params = derive_crr(inputs)
    out = {}
    t0 = time.time()
    for kind in (PayoffKind.ASIAN_PUT, PayoffKind.FIXED_LOOKBACK_PUT):
        req = ValuationRequest(inputs=inputs, params=params, kind=kind, workers=CORES, force_large=True)
        out[kind.value] = value_exact_parallel(req)
    dump("exact_paper.json", {"provenance": provenance({"wall_s": time.time() - t0}),
                              "N": 32, "S0": 20.0, "K": 100.0, "q": 0.06, "sigma": 3.0, "T": 1.0,
                              "u": params.u, "d": params.d, "p": float(params.up_probs[0]),
                              "published": {"asian-put": 82.115, "lookback-put": 93.196},
                              "values": out})


def batch_options(n_opts=4096, seed=0):
    rng = np.random.default_rng(seed)
    S0 = rng.uniform(50, 150, n_opts)
    m = rng.uniform(0.8, 1.2, n_opts)
    K = m * S0
    sigma = rng.uniform(0.1, 0.5, n_opts)
    r = rng.uniform(0.0, 0.08, n_opts)
    T = rng.uniform(0.25, 3.0, n_opts)
    return S0, K, sigma, r, T


def gen_batch():
    N = 24
    S0, K, sigma, r, T = batch_options()
    idx = list(range(0, 4096, 256)) + [4095]
    out = []
    t0 = time.time()
    for i in idx:
        params = classic_crr(N, float(sigma[i]), float(r[i]), float(T[i]))
        v = asian_call_route(params, float(S0[i]), float(K[i]), float(r[i]), float(T[i]), N, workers=CORES)
        out.append({"index": i, "S0": float(S0[i]), "K": float(K[i]), "sigma": float(sigma[i]),
                    "r": float(r[i]), "T": float(T[i]), "u": params.u, "d": params.d,
                    "p": float(params.up_probs[0]), "asian_call": v})
    dump("exact_batch.json", {"provenance": provenance({"wall_s": time.time() - t0}),
                              "config": "BASELINE configs[4]", "N": N, "n_options": 4096,
                              "rule": "rng=default_rng(0); S0=U(50,150); m=U(.8,1.2); K=m*S0; sigma=U(.1,.5); r=U(0,.08); T=U(.25,3)",
                              "options": out})


def gen_mc():
    """Reference MC statistics (numpy Philox stream; parity is statistical)."""
    out = {"provenance": provenance(), "studies": []}
    # DESK tree of tests/test_mc.py:29-30 (beta-CRR, N=12)
    desk = MarketInputs(S0=20.0, K=100.0, q=0.06, sigma=3.0, T=1.0, N=12)
    dp = derive_crr(desk)
    for kind in (PayoffKind.ASIAN_PUT, PayoffKind.FIXED_LOOKBACK_PUT):
        req = ValuationRequest(inputs=desk, params=dp, kind=kind)
        exact = value_exact_serial(req)
        rec = {"tree": "desk", "N": 12, "kind": kind.value, "exact": exact, "runs": {}}
        for tag, est, cfg in [("basic", estimate_basic, McConfig(R=128, seed=31, reps=400)),
                              ("pmc", estimate_partitioned, McConfig(R=128, M=4, seed=37, reps=400)),
                              ("pmc-equal", estimate_partitioned_equal, McConfig(R=32, M=4, seed=41, reps=400)),
                              ("smc", estimate_shared, McConfig(R=128, M=4, seed=43, reps=400))]:
            s = run_repetitions(est, req, cfg)
            rec["runs"][tag] = {"R": cfg.R, "M": cfg.M, "reps": cfg.reps, "mean_value": s.mean_value,
                                "mean_variance": s.mean_variance, "empirical_variance": s.empirical_variance}
        out["studies"].append(rec)
    # variance-reduction ratios, Asian call (sign-flip route), classic CRR, k=12
    for N in (32, 62):
        params = classic_crr(N, 0.2, 0.05, 1.0)
        inputs = SimpleNamespace(S0=-100.0, K=-100.0, q=0.05, T=1.0, N=N)
        req = ValuationRequest(inputs=inputs, params=params, kind=PayoffKind.ASIAN_PUT)
        reps = 10
        R_total = 1 << 18
        b = run_repetitions(estimate_basic, req, McConfig(R=R_total, seed=7, reps=reps))
        e = run_repetitions(estimate_partitioned_equal, req, McConfig(R=R_total >> 12, M=4096, seed=7, reps=reps))
        p = run_repetitions(estimate_partitioned, req, McConfig(R=R_total, M=4096, seed=7, reps=reps))
        out["studies"].append({"tree": "classic", "N": N, "kind": "asian-call", "S0": 100.0, "K": 100.0,
                               "r": 0.05, "sigma": 0.2, "T": 1.0, "k": 12, "R_total": R_total, "reps": reps,
                               "basic": {"mean_value": b.mean_value, "mean_variance": b.mean_variance},
                               "pmc-equal": {"mean_value": e.mean_value, "mean_variance": e.mean_variance},
                               "pmc": {"mean_value": p.mean_value, "mean_variance": p.mean_variance},
                               "ratio_basic_over_equal": b.mean_variance / e.mean_variance,
                               "ratio_basic_over_pmc": b.mean_variance / p.mean_variance})
    dump("mc_reference.json", out)


def gen_cli():
    """Reference CLI / bench-harness outputs: report values of the exact
    methods and the bench CSV / table rendering of fixed records."""
    from binpaths import cli
    from binpaths.bench import BenchRecord, records_to_csv, records_to_tables
    import contextlib
    import io

    def run(*argv):
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            code = cli.main(list(argv))
        return code, buf.getvalue()

    desk = ["--S0", "20", "--K", "100", "--q", "0.06", "--sigma", "3.0", "--T", "1"]
    price = []
    for method in ("exact", "exact-serial", "leaf"):
        for payoff in ("euro-call", "euro-put", "asian-put", "lookback-put"):
            if method == "leaf" and payoff in ("asian-put", "lookback-put"):
                continue
            for N, workers in ((12, 1), (12, 4), (16, 3)):
                argv = ["price", "--method", method, "--payoff", payoff, "--N", str(N), "--workers", str(workers)]
                code, out = run(*argv, *desk)
                rep = json.loads(out)
                rep.pop("wall_seconds")
                price.append({"argv": argv + desk, "code": code, "report": rep})
    code, out = run("price", "--method", "exact", "--payoff", "euro-put", "--S0", "4", "--K", "5", "--q", "0",
                    "--sigma", "0.30", "--T", "1", "--N", "2", "--override-u", "2", "--override-p", "0.5")
    hand = json.loads(out)
    hand.pop("wall_seconds")
    recs = [BenchRecord(n=n, m=m, wall_seconds=w, speedup=s, efficiency=s / m, baseline_m=b)
            for n, m, w, s, b in ((8, 1, 0.5, 1.0, 1), (8, 2, 0.26, 1.0 / 0.52, 1), (8, 4, 0.1301, 0.5 / 0.1301, 1),
                                  (10, 2, 1.25, 2.0, 2), (10, 4, 0.7, 2.5 / 0.7, 2))]
    fmt = {"records": [r.__dict__ for r in recs], "csv": records_to_csv(recs), "tables": records_to_tables(recs)}
    dump("cli_reference.json", {"provenance": provenance(), "price": price, "hand_example": hand, "bench_format": fmt})


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["small"]
    table = {"small": gen_small, "config1": gen_config1, "config2": gen_config2,
             "config3": gen_config3, "paper": gen_paper, "batch": gen_batch, "mc": gen_mc,
             "cli": gen_cli}
    for w in which:
        t = time.time()
        table[w]()
        print(w, "done in", round(time.time() - t, 1), "s", flush=True)
