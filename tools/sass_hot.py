"""Summarise an `ncu --page source --csv --print-source sass` export: stall
samples by opcode and the hottest instructions (development tool)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))[1:]
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
agg, tot, top = collections.Counter(), 0.0, []
for i, r in enumerate(rows[1:]):
    try:
        v = float(r[si] or 0)
    except ValueError:
        continue
    toks = r[src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    agg[op.split(".")[0]] += v
    tot += v
    top.append((v, i, r[src].strip()[:80]))
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 15):
    print(f"{k:12s} {v / tot * 100:6.2f}%")
print("--- hottest")
for v, i, s in sorted(top, reverse=True)[: int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{v / tot * 100:6.2f}%  #{i:5d}  {s}")
