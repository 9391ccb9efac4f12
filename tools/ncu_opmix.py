"""Per-opcode executed warp instructions of one ncu --set full capture (its
SASS source page), normalised per 32 leaf tests (one warp-wide leaf test).

  python tools/ncu_opmix.py <report.ncu-rep> <leaf_tests>
FP64-pipe opcodes (DSETP, DFMA, DADD, DMUL, DMNMX, MUFU.RCP64H, F2F/I2F .F64)
are summed separately: their count per leaf test is the 'executed FP64-pipe
ops per leaf test' bench.py's bounded roofline fraction uses."""
import collections
import csv
import io
import json
import subprocess
import sys

FP64 = ("DSETP", "DFMA", "DADD", "DMUL", "DMNMX", "MUFU.RCP64H", "F2F.F64", "I2F.F64", "F2I.F64", "DSET")


def opmix(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    agg = collections.Counter()
    for r in rows[2:]:
        tok = r[i_src].split()
        if not tok:
            continue
        op = tok[1] if tok[0].startswith("@") else tok[0]
        agg[op] += float(r[i_ex] or 0)
    return agg


def main():
    rep, leaf_tests = sys.argv[1], float(sys.argv[2])
    agg = opmix(rep)
    per = 32.0 / leaf_tests
    fp64 = sum(v for op, v in agg.items() if op.startswith(FP64))
    total = sum(agg.values())
    by_root = collections.Counter()
    for op, v in agg.items():
        by_root[op.split(".")[0]] += v
    print(json.dumps({"report": rep, "leaf_tests": leaf_tests, "warp_inst_per_32_leaf_tests": total * per,
                      "fp64_pipe_warp_inst_per_32_leaf_tests": fp64 * per,
                      "by_opcode_per_32_leaf_tests": {k: round(v * per, 4) for k, v in by_root.most_common(16)}},
                     indent=1))


if __name__ == "__main__":
    main()
