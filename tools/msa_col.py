"""Time MSA column attention (bias-free plus mask; the attended axis is N_seq) fwd+bwd on cuda:0.

  python tools/msa_col.py [--rows 384] [--L 512] [--H 8] [--D 32] [--iters 20]
Rows are the N_res columns of the MSA, L = N_seq. Prints TFLOP/s (14*B*H*L^2*D convention).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2310_04610_b200 as E

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=384)
ap.add_argument("--L", type=int, default=512)
ap.add_argument("--H", type=int, default=8)
ap.add_argument("--D", type=int, default=32)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(7)
u = lambda *s: (torch.rand(*s, generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
q, k, v, do = (u(1, a.rows, a.L, a.H, a.D) for _ in range(4))
m = torch.rand(1, a.rows, 1, 1, a.L, generator=g, device=dev) < 0.1
m[..., 0] = False
b1 = torch.where(m, -1e9, 0.0).to(torch.bfloat16)


def step():
    o, lse = E.evoformer_attention_forward(q, k, v, b1)
    E.evoformer_attention_backward(do, q, k, v, o, lse, b1, None)


for _ in range(3):
    step()
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(a.iters):
    step()
t1.record()
torch.cuda.synchronize()
ms = t0.elapsed_time(t1) / a.iters
fl = 14.0 * a.rows * a.H * a.L * a.L * a.D
print(f"msa_col rows={a.rows} L={a.L} H={a.H} D={a.D}: {ms:.3f} ms/step  {fl / ms / 1e9:.1f} TFLOP/s  path={E.resolved_path(q, b1, None)}")
