"""Aggregate ncu source-page (SASS) warp-stall samples by opcode (developer tool).
    python tools/ncu_sass_stalls.py src.csv"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS = hdr.index("Source"); iW = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: hdr.index(c) for c in cols}
by_op, by_op_ex, tot = Counter(), Counter(), 0
reasons = {}
for r in rows[2:]:
    if len(r) <= iW or not r[iW]:
        continue
    op = r[iS].split()[0] if r[iS].split() else "?"
    if op.startswith("@"):
        op = r[iS].split()[1]
    op = op.split(".")[0]
    w = float(r[iW] or 0)
    by_op[op] += w
    by_op_ex[op] += float(r[iE] or 0)
    tot += w
    rr = reasons.setdefault(op, Counter())
    for c in cols:
        try:
            rr[c] += float(r[idx[c]] or 0)
        except ValueError:
            pass
for op, w in by_op.most_common(18):
    top = ", ".join(f"{k[6:]}={v/max(w,1)*100:.0f}%" for k, v in reasons[op].most_common(3))
    print(f"{op:10s} {100*w/tot:5.1f}% samples  inst {by_op_ex[op]:.3g}  [{top}]")
