"""Multi-GPU check of the row-sharding launcher (torchrun, one rank per GPU):
the in-kernel NVLS dBias2 reduction (multicast) against a local backward + NCCL all-reduce.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_check.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("EVO_MULTICAST", "1")  # exercise the in-kernel NVLS reduction
import torch
import torch.distributed as dist

import bench
import paper_2310_04610_b200 as E
from paper_2310_04610_b200 import sharded

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=dev)
cfg = (1, 96, 384, 8, 32, "bf16", "check")
q, k, v, do, b1, b2 = (t.to(dev) for t in bench.make_inputs(cfg, (0, 96)))
mc = sharded._multicast_dbias2(b2, None)
r = sharded.sharded_fwd_bwd(q, k, v, do, b1, b2)
o, lse = E.evoformer_attention_forward(q, k, v, b1, b2)
_, _, _, _, ref = E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2)
dist.all_reduce(ref)
torch.cuda.synchronize()
err = ((r.dbias2 - ref).abs().max() / ref.abs().max()).item()
print(f"rank {rank}: multicast={'yes' if mc is not None else 'no'} dbias2 max rel diff vs NCCL all-reduce {err:.2e}",
      flush=True)
assert err < 1e-5, err
dist.destroy_process_group()
