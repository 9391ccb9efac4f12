"""Executed-instruction mix of one kernel from an ncu report's source page:
opcode, executed warp instructions, per warp-level leaf test, stall samples.

  python tools/sass_mix.py <report.ncu-rep> <leaf tests per launch> [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, leaves = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
cnt, stall = collections.Counter(), collections.Counter()
for row in rows[2:]:
    if len(row) <= ie or not row[src].strip():
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", row[src].strip()).split()[0]
    cnt[op] += int(row[ie] or 0)
    stall[op] += int(row[st] or 0)
wl = leaves / 32
tot = sum(cnt.values())
print(f"{'opcode':22s} {'executed':>14s} {'/warp-leaf':>10s} {'stalls':>8s}")
for k, v in cnt.most_common(top):
    print(f"{k:22s} {v:14d} {v / wl:10.3f} {stall[k]:8d}")
print(f"{'total':22s} {tot:14d} {tot / wl:10.3f} {sum(stall.values()):8d}")
