import sys, time, torch
sys.path.insert(0, "/root/repo")
import bench
import paper_2310_04610_b200 as E
from paper_2310_04610_b200.sharded import sharded_fwd_bwd
E.set_numeric_checks(False)
cfg = bench.CONFIGS["c4"]
q, k, v, do, b1, b2 = (t.cuda() for t in bench.make_inputs(cfg, (0, 512), pin=True))
def run(n, label, fn):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record()
    for _ in range(n): fn()
    t1 = time.perf_counter(); b.record(); torch.cuda.synchronize()
    print(label, "gpu ms/step", round(a.elapsed_time(b) / n, 4), "host enqueue ms/step", round((t1 - t0) * 1e3 / n, 4), flush=True)
run(20, "sharded", lambda: sharded_fwd_bwd(q, k, v, do, b1, b2))
def raw():
    o, lse = E.evoformer_attention_forward(q, k, v, b1, b2)
    E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2)
run(20, "raw", raw)
with bench.ClockSampler(0):
    run(20, "sharded+clock", lambda: sharded_fwd_bwd(q, k, v, do, b1, b2))
