"""Executed warp instructions of one kernel per CUDA source line: joins an ncu
capture's SASS page (per-instruction counts, in address order) with
nvdisasm -g line info of the same cubin (same instruction order).
  python tools/sass_by_line.py <report.ncu-rep> <object.o> <mangled-name substring> [top]"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, obj, name = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ia = hdr.index("Instructions Executed")
execs = [int(r[ia]) for r in data]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
# walk the function's section: track the current "//## File ..., line N" and inline chain
lines, cur, infn = [], None, False
for ln in dis.splitlines():
    if ln.startswith("//--------------------- .text."):
        infn = name in ln
        continue
    if not infn:
        continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)), "inlined" in m.group(3))
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", ln):
        lines.append(cur)
if len(lines) != len(execs):
    print(f"warning: {len(lines)} disassembled instructions vs {len(execs)} in the capture", file=sys.stderr)
agg = collections.Counter()
for loc, e in zip(lines, execs):
    agg[(loc[0], loc[1]) if loc else ("?", 0)] += e
tot = sum(execs)
print(f"total {tot} warp instructions")
for (f, l), c in agg.most_common(top):
    print(f"{100 * c / tot:5.1f}%  {f}:{l}")
