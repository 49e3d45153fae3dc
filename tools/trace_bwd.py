"""Print the CTA-0 timeline of one backward launch, steps 100..163 (bring-up aid; see
evo_attn_debug_set_trace_bwd)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2310_04610_b200 as E
from paper_2310_04610_b200 import _native as N

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = bench.CONFIGS[args[0] if args else "c4"]
dev = torch.device("cuda:0")
q, k, v, do, b1, b2 = (t.to(dev) for t in bench.make_inputs(cfg, (0, cfg[1])))
if "--nobias" in sys.argv:
    b1 = b2 = None
if "--nob1" in sys.argv:
    b1 = None
o, lse = E.evoformer_attention_forward(q, k, v, b1, b2)
for _ in range(2):
    E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2)
buf = torch.zeros(12 * 64, dtype=torch.int64, device=dev)
lib = N.load()
lib.evo_attn_debug_set_trace_bwd.argtypes = [ctypes.c_void_p]
lib.evo_attn_debug_set_trace_bwd(buf.data_ptr())
E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2)
torch.cuda.synchronize()
lib.evo_attn_debug_set_trace_bwd(None)
t = buf.view(12, 64).cpu().tolist()
t0 = min(x for row in t for x in row if x > 0)
names = ["S_issue", "S_seen", "Pds_wg0", "Pds_wg3", "Grads", "Dq_seen", "Dq_out", "Q_full", "ProdQ", "K_full", "GradsSt", "S_done"]
if "--phase" in sys.argv:  # library built with -DEVO_BWD_PHASE_TRACE=1
    names[7:12] = ["ph_qfull", "ph_ldtm", "ph_math", "ph_sts", "ph_waits"]
print("step " + " ".join(f"{n:>9s}" for n in names))
for s in range(64):
    print(f"{s + 100:4d} " + " ".join(f"{(t[e][s] - t0) if t[e][s] else -1:9d}" for e in range(12)))
