"""Hot SASS instructions (stall samples, top reasons) from an ncu source-page CSV:
python scripts/sass_hot.py gpurun_out/src_<kernel>_sass.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
R = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
st = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
samp = lambda r: int(r["Warp Stall Sampling (All Samples)"] or 0)
tot = sum(samp(r) for r in R)
reasons = collections.Counter()
ops = collections.Counter()
for r in R:
    for k in st:
        reasons[k[6:]] += int(r[k] or 0)
    src = r["Source"].strip().split()
    op = (src[1] if src and src[0].startswith("@") and len(src) > 1 else (src[0] if src else "")).split(".")[0]
    ops[op] += samp(r)
print("samples", tot, "instrs executed", sum(int(r["Instructions Executed"] or 0) for r in R))
print("reasons", [(k, round(v / tot * 100, 1)) for k, v in reasons.most_common(9)])
print("ops", [(k, round(v / tot * 100, 1)) for k, v in ops.most_common(14)])
for r in sorted(R, key=lambda r: -samp(r))[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    d = sorted(((int(r[k] or 0), k[6:]) for k in st if int(r[k] or 0)), reverse=True)[:3]
    print(r["Address"][-5:], samp(r), r["Source"].strip()[:48], d)
