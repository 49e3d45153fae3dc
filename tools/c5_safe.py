import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04610_b200 as E
cfgs = {"c5": (1, 2048, 2048, 4, 32), "c4": (1, 512, 384, 8, 32)}
for name, (Bo, Nr, L, H, D) in cfgs.items():
    g = torch.Generator(device="cuda").manual_seed(7)
    u = lambda *s: (torch.rand(*s, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    q, k, v, do = (u(Bo, Nr, L, H, D) for _ in range(4))
    b2 = u(Bo, 1, H, L, L)
    b1 = torch.zeros(Bo, Nr, 1, 1, L, device="cuda", dtype=torch.bfloat16)
    o, lse = E.evoformer_attention_forward(q, k, v, b1, b2, check_numerics=False)
    def t(chk, n=3):
        for _ in range(2): E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2, check_numerics=chk)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(n): E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2, check_numerics=chk)
        b.record(); torch.cuda.synchronize()
        return a.elapsed_time(b) / n
    print(name, "bwd unchecked", round(t(False), 3), "checked (SAFE kernel)", round(t(True), 3), flush=True)
