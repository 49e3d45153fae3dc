"""Print the main-kernel launch times of each A/B variant csv: python tools/ab_parse.py v1 v2 ..."""
import csv
import sys

for v in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f"gpurun_out/abm_{v}.csv")) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    main = [float(r[vi].replace(",", "")) / 1e3 for r in rows[1:] if "bwd_kernel" in r[ki] or "fwd_kernel" in r[ki]]
    print(f"{v:8s}", " ".join(f"{t:.1f}" for t in main[-3:]))
