import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2310_04610_b200 as E
from tests.util import make_inputs
E.set_numeric_checks(False)
shape = (2, 5, 256, 2, 32)
inp = [None if a is None else torch.tensor(a, dtype=torch.bfloat16, device="cuda") for a in make_inputs(*shape, seed=31)]
q, k, v, do, b1, b2 = inp
o, lse = E.evoformer_attention_forward(q, k, v, b1, b2)
os.environ.pop("EVO_BWD_WINDOW_ROWS", None)
ref = E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2)
for wr in ["1", "2", "3", "4"]:
    os.environ["EVO_BWD_WINDOW_ROWS"] = wr
    got = E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2)
    torch.cuda.synchronize()
    a, b = got[0].float(), ref[0].float()
    d = (a - b).abs().amax(dim=(3, 4))  # per (ob, n, i)
    per_row = d.amax(dim=2)
    print("win", wr, "dq err per (ob,n):", [[round(float(x), 3) for x in r] for r in per_row], flush=True)
    bad = (d > 1e-3).nonzero()
    if len(bad):
        print("   bad query rows of (ob=0,n=0):", sorted(set(int(x[2]) for x in bad if x[0] == 0 and x[1] == 0))[:20], "count", len(bad))
    print("   ratio got/ref rows (0,0,0..3):", [round(float((a[0, 0, i] / b[0, 0, i]).median()), 3) for i in range(4)])
