import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2310_04610_b200 as E
L, H, cz = 384, 8, 128
z = torch.randn(1, L, L, cz, device="cuda").to(torch.bfloat16)
g, b = torch.ones(cz, device="cuda"), torch.zeros(cz, device="cuda")
w = torch.randn(H, cz, device="cuda") / cz ** 0.5
db2 = torch.randn(1, 1, H, L, L, device="cuda")
E.pair_bias_forward(z, g, b, w); E.pair_bias_backward(db2, z, g, b, w)
torch.cuda.synchronize(); print("ok")
