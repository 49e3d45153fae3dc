"""Summarise an ncu --page source --csv --print-source=sass dump: top instructions by stall samples."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
data = [dict(zip(h, r)) for r in rows[hdr_i + 1:] if len(r) == len(h)]
tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total samples", tot)
top = sorted(data, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for d in top:
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f'{s / tot * 100:5.1f}% {d["Address"]:>6} {d["Source"][:90]}')
# opcode histogram weighted by samples
c = Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"] else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    c[op.split(".")[0]] += float(d["Warp Stall Sampling (All Samples)"] or 0)
print({k: round(v / tot * 100, 1) for k, v in c.most_common(15)})
