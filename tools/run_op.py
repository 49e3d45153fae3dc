"""Run the hot-path op at a BASELINE config a few times (for ncu / sanitizer captures).

  python tools/run_op.py --config c4 --what fwd|bwd|both --iters 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2310_04610_b200 as E

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--what", default="both")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--path", default="auto")
ap.add_argument("--shape", default=None, help="Bo,N,L,H,D (bf16) instead of a config")
a = ap.parse_args()
E.set_numeric_checks(False)
if a.shape:
    Bo, Nr, L, H, D = map(int, a.shape.split(","))
    cfg = (Bo, Nr, L, H, D, "bf16", "shape " + a.shape)
else:
    cfg = bench.CONFIGS[a.config]
dev = torch.device("cuda:0")
q, k, v, do, b1, b2 = (t.to(dev) for t in bench.make_inputs(cfg, (0, cfg[1])))
o, lse = E.evoformer_attention_forward(q, k, v, b1, b2, path=a.path)
for _ in range(a.iters):
    if a.what in ("fwd", "both"):
        o, lse = E.evoformer_attention_forward(q, k, v, b1, b2, path=a.path)
    if a.what in ("bwd", "both"):
        E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2, need_dbias1=False, path=a.path)
torch.cuda.synchronize()
print("ok", a.shape or a.config, a.what, E.resolved_path(q, b1, b2, a.path))
