import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04610_b200 as E
Bo, Nr, L, H, D = 1, 2048, 2048, 4, 32
g = torch.Generator(device="cuda").manual_seed(7)
u = lambda *s: (torch.rand(*s, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
q, k, v, do = (u(Bo, Nr, L, H, D) for _ in range(4))
b2 = u(Bo, 1, H, L, L)
b1 = torch.zeros(Bo, Nr, 1, 1, L, device="cuda", dtype=torch.bfloat16)
o, lse = E.evoformer_attention_forward(q, k, v, b1, b2, check_numerics=False)
E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2, check_numerics=False)
torch.cuda.synchronize()
