"""Time the fused pair-bias projection (LN(z)·W → bias2 [Bo, 1, H, L, L]; backward from dBias2 in that
layout) against the torch composition OpenFold runs (layer_norm → linear → permute → contiguous; its
autograd backward). CUDA events, L2-sized inputs at C4 / C5 pair shapes.
  python tools/pair_bias_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2310_04610_b200 as E


def t(fn, n=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


res = {}
for name, (L, H) in {"c4": (384, 8), "c5": (2048, 4)}.items():
    cz = 128
    z = torch.randn(1, L, L, cz, device="cuda").to(torch.bfloat16)
    g, b = torch.ones(cz, device="cuda"), torch.zeros(cz, device="cuda")
    w = torch.randn(H, cz, device="cuda") / cz ** 0.5
    db2 = torch.randn(1, 1, H, L, L, device="cuda")
    fwd = t(lambda: E.pair_bias_forward(z, g, b, w))
    bwd = t(lambda: E.pair_bias_backward(db2, z, g, b, w))
    lnm = torch.nn.LayerNorm(cz).cuda().to(torch.bfloat16)
    lin = torch.nn.Linear(cz, H, bias=False).cuda().to(torch.bfloat16)

    def torch_fwd():
        return lin(lnm(z)).permute(0, 3, 1, 2).unsqueeze(1).contiguous()

    zt = z.clone().requires_grad_()

    def torch_fb():
        out = lin(lnm(zt)).permute(0, 3, 1, 2).unsqueeze(1).contiguous()
        out.backward(db2.to(torch.bfloat16))

    tf = t(torch_fwd)
    tfb = t(torch_fb)
    zb = z.numel() * 2
    res[name] = {"L": L, "H": H, "c_z": cz, "fused_fwd_ms": fwd, "fused_bwd_ms": bwd,
                 "fused_fwd_gbs": (zb + H * L * L * 2) / fwd / 1e6,
                 "fused_bwd_gbs": (2 * zb + H * L * L * 4) / bwd / 1e6,
                 "torch_fwd_ms": tf, "torch_fwd_bwd_ms": tfb}
print(json.dumps(res, indent=1))
