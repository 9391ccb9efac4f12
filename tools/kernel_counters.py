"""Write the dominant kernel's per-launch counters from an ncu --set full
capture into profiles/r2_kernel_counters.json (read by bench.py's roofline).

  python tools/kernel_counters.py <workload> <report.ncu-rep> <leaf_tests_per_launch>
"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_opmix import FP64, opmix  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                   "r2_kernel_counters.json")


def main():
    workload, rep, leaf_tests = sys.argv[1], sys.argv[2], float(sys.argv[3])
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    m = dict(zip(rows[0], rows[2]))

    def num(k):
        v = m.get(k)
        return float(str(v).replace(",", "")) if v not in (None, "") else None

    agg = opmix(rep)
    per = 32.0 / leaf_tests
    fp64 = sum(v for op, v in agg.items() if op.startswith(FP64))
    entry = {
        "source": os.path.basename(rep),
        "kernel": m.get("Kernel Name", "")[:80],
        "duration_us": num("gpu__time_duration.sum") / 1e3,  # base unit: ns
        "dram_bytes_read": num("dram__bytes_read.sum"),
        "dram_bytes_write": num("dram__bytes_write.sum"),
        "fp64_pipe_active_pct": num("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "fma_pipe_active_pct": num("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        "alu_pipe_active_pct": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "warp_inst_per_32_leaf_tests": sum(agg.values()) * per,
        "fp64_pipe_ops_per_leaf_test": fp64 * per,
        "local_loads": num("smsp__sass_inst_executed_op_local_ld.sum"),
        "local_stores": num("smsp__sass_inst_executed_op_local_st.sum"),
        "registers": num("launch__registers_per_thread"),
    }
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data[workload] = entry
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1)
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main()
