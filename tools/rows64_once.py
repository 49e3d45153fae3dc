"""One forward + backward call of C4 on 64 rows (the per-rank work of an 8-GPU strong-scaling run)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2310_04610_b200 as E

E.set_numeric_checks(False)
cfg = bench.CONFIGS["c4"]
q, k, v, do, b1, b2 = (x.cuda() for x in bench.make_inputs(cfg, (0, int(sys.argv[1]) if len(sys.argv) > 1 else 64)))
for _ in range(3):
    o, lse = E.evoformer_attention_forward(q, k, v, b1, b2)
    E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2)
torch.cuda.synchronize()
print("ok")
