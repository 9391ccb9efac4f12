"""Opcode mix of one ncu capture's hottest kernel (source page): warp
instructions per unit of work and stall share per opcode.
  python tools/sass_hot.py <report.ncu-rep> <units, e.g. warp-draws>"""
import collections, csv, io, subprocess, sys
rep, units = sys.argv[1], float(eval(sys.argv[2]))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ia, iss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ia]) for r in data); tots = sum(int(r[iss]) for r in data)
mix, smix = collections.Counter(), collections.Counter()
for r in data:
    t = r[1].split()
    op = t[1] if t[0].startswith("@") else t[0]
    op = ".".join(op.split(".")[:2]) if op.startswith(("IMAD", "LOP3", "IADD")) else op.split(".")[0]
    mix[op] += int(r[ia]); smix[op] += int(r[iss])
print(f"total {tot} warp instructions, {tot / units:.1f} per unit")
for op, c in mix.most_common(30):
    print("%-12s %5.1f%% inst  %5.1f%% stall  per unit %.1f" % (op, 100 * c / tot, 100 * smix[op] / tots, c / units))
