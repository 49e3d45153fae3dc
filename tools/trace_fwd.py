"""Print the CTA-0 timeline of one forward launch (bring-up aid; see evo_attn_debug_set_trace)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2310_04610_b200 as E
from paper_2310_04610_b200 import _native as N

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
dev = torch.device("cuda:0")
q, k, v, do, b1, b2 = (t.to(dev) for t in bench.make_inputs(cfg, (0, cfg[1])))
for _ in range(3):
    E.evoformer_attention_forward(q, k, v, b1, b2)
buf = torch.zeros(12 * 64, dtype=torch.int64, device=dev)
lib = N.load()
lib.evo_attn_debug_set_trace.argtypes = [ctypes.c_void_p]
lib.evo_attn_debug_set_trace(buf.data_ptr())
E.evoformer_attention_forward(q, k, v, b1, b2)
torch.cuda.synchronize()
lib.evo_attn_debug_set_trace(None)
t = buf.view(12, 64).cpu().tolist()
t0 = min(x for row in t for x in row if x > 0)
names = ["Vload", "S_issue", "S_seen", "P_wg0", "P_wg1", "PV_issue", "RowEnd", "RowStart", "Pfull_ok", "Vfull_ok", "Kload", "Kfull_ok"]
print("tile " + " ".join(f"{n:>9s}" for n in names))
for tile in range(40):
    print(f"{tile:4d} " + " ".join(f"{(t[e][tile] - t0) if t[e][tile] else -1:9d}" for e in range(12)))
