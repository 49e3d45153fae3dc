"""Per-rank cost of C4 at the row counts strong scaling gives each rank (512 / N rows for N = 1..8):
forward and backward call times on one GPU, against the ideal 1/N of the full-problem time.
  python tools/rows_scan.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2310_04610_b200 as E

E.set_numeric_checks(False)
cfg = bench.CONFIGS["c4"]


def t(fn, n=30):
    for _ in range(5):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


full = None
for n in (1, 2, 4, 8, 16):
    rows = cfg[1] // n
    q, k, v, do, b1, b2 = (x.cuda() for x in bench.make_inputs(cfg, (0, rows)))
    o, lse = E.evoformer_attention_forward(q, k, v, b1, b2)
    tf = t(lambda: E.evoformer_attention_forward(q, k, v, b1, b2))
    tb = t(lambda: E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2))
    full = full or (tf + tb)
    print(f"N={n:2d} rows/rank={rows:3d}: fwd {tf:.4f} bwd {tb:.4f} ms, step {tf + tb:.4f} (ideal {full / n:.4f}, "
          f"{full / n / (tf + tb):.0%} of linear)")
