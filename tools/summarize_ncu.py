"""Summarise ncu captures into a markdown table (used to write profiles/).

  python tools/summarize_ncu.py <report.ncu-rep> [...]   -> key metrics per kernel
  python tools/summarize_ncu.py --launches <launches.csv>  -> per-kernel share of a run
"""
import csv
import collections
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration", 1),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (GHz)", 1),
    ("launch__registers_per_thread", "registers/thread", 1),
    ("launch__grid_size", "grid", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %", 1),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %", 1),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %", 1),
    ("smsp__inst_executed.sum", "warp instructions", 1),
    ("dram__bytes_read.sum", "DRAM read", 1),
    ("dram__bytes_write.sum", "DRAM write", 1),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per warp instruction (divergence)", 1),
    ("smsp__sass_average_branch_targets_threads_uniform.pct", "uniform branch targets %", 1),
    ("smsp__sass_inst_executed_op_local_ld.sum", "local (spill) loads, warp inst", 1),
    ("smsp__sass_inst_executed_op_local_st.sum", "local (spill) stores, warp inst", 1),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not_selected", 1),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe", 1),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio", 1),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait", 1),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard", 1),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    hdr = [h + (f" [{u}]" if u and u not in ("%", "inst", "warp", "register/thread", "cycle") else "")
           for h, u in zip(hdr, units)]
    return hdr, rows[2:]


def summarize(reps):
    print("| metric | " + " | ".join(r.split("/")[-1] for r in reps) + " |")
    print("|---|" + "---|" * len(reps))
    cols = [raw(r) for r in reps]
    names = []
    for hdr, data in cols:
        names.append(data[0][hdr.index("Kernel Name")][:48])
    print("| kernel | " + " | ".join(names) + " |")
    for key, label, scale in KEYS:
        vals = []
        for hdr, data in cols:
            try:
                col = next(i for i, h in enumerate(hdr) if h == key or h.startswith(key + " ["))
                if col is not None and "[" in hdr[col] and vals == []:
                    pass
                v = float(data[0][col].replace(",", "")) * scale
                u = hdr[col][hdr[col].find("[") + 1:-1] if "[" in hdr[col] else ""
                vals.append((f"{v:,.3g}" if abs(v) < 1e4 else f"{v:,.0f}") + (f" {u}" if u else ""))
            except (ValueError, IndexError, StopIteration):
                vals.append("n/a")
        print(f"| {label} | " + " | ".join(vals) + " |")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        try:
            agg[re.sub(r"\(.*", "", r[ki])[:70]].append(float(r[vi].replace(",", "")))
        except ValueError:
            pass
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | total (us) | share | mean (us) |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% | {sum(v) / len(v) / 1e3:.1f} |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        summarize(sys.argv[1:])
