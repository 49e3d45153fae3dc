"""A/B timing of library variants on one box: python tools/ab_time.py v1 v2 ... [--config c4] [--rounds 3].
Each variant lib/libevoattn_<v>.so is timed in its own process (forward call, backward call, CUDA
events, 30 iterations after warm-up), alternating rounds so box drift hits every variant alike."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2310_04610_b200", "lib")

CHILD = r'''
import json, sys, torch
sys.path.insert(0, ROOT)
import bench
import paper_2310_04610_b200 as E
cfg = bench.CONFIGS[CFG]
Bo, Nr, L, H, D, dt, _ = cfg
g = torch.Generator(device="cuda").manual_seed(7)
u = lambda *s: (torch.rand(*s, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
q, k, v, do = (u(Bo, Nr, L, H, D) for _ in range(4))
m = torch.rand(Bo, Nr, 1, 1, L, generator=g, device="cuda") < 0.1
m[..., 0] = False
b1 = torch.where(m, -1e9, 0.0).to(torch.bfloat16)
b2 = u(Bo, 1, H, L, L)
kw = {"check_numerics": False} if "check_numerics" in E.evoformer_attention_forward.__code__.co_varnames else {}
def t(fn, n=30):
    for _ in range(3): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
o, lse = E.evoformer_attention_forward(q, k, v, b1, b2, **kw)
f = t(lambda: E.evoformer_attention_forward(q, k, v, b1, b2, **kw))
bw = t(lambda: E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2, **kw))
print(json.dumps({"fwd": round(f, 4), "bwd": round(bw, 4), "sum": round(f + bw, 4)}))
'''

args = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = "c4"
rounds = 3
for i, a in enumerate(sys.argv):
    if a == "--config":
        cfg = sys.argv[i + 1]
    if a == "--rounds":
        rounds = int(sys.argv[i + 1])
variants = [a for a in args if a not in (cfg, str(rounds))]
res = {v: [] for v in variants}
for r in range(rounds):
    for v in variants:
        env = dict(os.environ, EVO_LIB=os.path.join(LIB, f"libevoattn_{v}.so"))
        out = subprocess.run([sys.executable, "-c", CHILD.replace("ROOT", repr(ROOT)).replace("CFG", repr(cfg))],
                             env=env, capture_output=True, text=True, timeout=300)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        print(v, line, flush=True)
        try:
            res[v].append(json.loads(line))
        except Exception:
            pass
for v, xs in res.items():
    if xs:
        print(f"{v:10s} fwd {min(x['fwd'] for x in xs):.4f} bwd {min(x['bwd'] for x in xs):.4f} "
              f"sum {min(x['sum'] for x in xs):.4f} (min of {len(xs)})")
