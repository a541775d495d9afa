"""Per-source-line instruction counts / stall samples of one profiled kernel launch:
joins the ncu SASS page (gpurun_out/srcc_<K>_sass.csv, absolute addresses) with the
line table of the kernel in the built object (nvdisasm --print-line-info).
usage: python scripts/sass_lines.py <object.o> <mangled-kernel-name> <sass.csv> [top]"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

obj, fn, sass, top = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, cubin)], capture_output=True,
                     text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if l.startswith(".text." + fn + ":"))
where, table = "?", {}
for l in dis[start + 1:]:
    if l.startswith(".text.") or l.startswith("\t.section"):
        break
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m:
        where = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*)", l)
    if m:
        table[int(m.group(1), 16)] = (where, m.group(2).split(";")[0].strip())
rows = list(csv.reader(open(sass)))
hi = 0 if "Source" in rows[0] else 1
h = rows[hi]
R = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) == len(h)]
base = min(int(r["Address"], 16) for r in R)
by = collections.defaultdict(lambda: [0, 0, collections.Counter()])
tot_i = tot_s = 0
for r in R:
    off = int(r["Address"], 16) - base
    line, ins = table.get(off, ("?", ""))
    n = int(r["Instructions Executed"] or 0)
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    op = r["Source"].strip().split()
    op = (op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else "")).split(".")[0]
    by[line][0] += n
    by[line][1] += s
    by[line][2][op] += n
    tot_i += n
    tot_s += s
print(f"instructions {tot_i}  stall samples {tot_s}")
for line, (n, s, ops) in sorted(by.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * n / tot_i:5.1f}% instr {100 * s / max(tot_s, 1):5.1f}% stall  {line:22s} {dict(ops.most_common(5))}")
