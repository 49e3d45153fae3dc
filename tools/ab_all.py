"""Per-kernel times of every evo kernel in the A/B csvs: python tools/ab_all.py v1 v2 ..."""
import csv
import re
import sys
from collections import defaultdict

for v in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f"gpurun_out/abm_{v}.csv")) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        m = re.search(r"(\w+_kernel)", r[ki])
        if m and ("evo::" in r[ki] or "bk::" in r[ki]):
            agg[m.group(1)].append(float(r[vi].replace(",", "")) / 1e3)
    print(f"{v:8s}", "  ".join(f"{k}={sum(t[-3:]) / len(t[-3:]):.1f}" for k, t in agg.items()))
