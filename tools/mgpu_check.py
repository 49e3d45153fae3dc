"""Multi-GPU checks of the row-sharding launcher (torchrun, one rank per GPU, NCCL):
  1. strong sharding of one problem (rows split over ranks): every rank's O / dQ / dK / dV rows are
     bit-identical to the single-GPU run of the whole problem, and the all-reduced dBias2 equals the
     single-GPU dBias2 up to fp32 summation order (blocking and asynchronous all-reduce);
  2. the 16-bit dBias2 path (conversion fused into the reduction) against the fp32 sum;
  3. the in-kernel NVLS dBias2 reduction (EVO_MULTICAST=1, multimem.red through an NVSwitch multicast
     mapping) against the NCCL all-reduce, where symmetric memory with multicast is available.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_check.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import bench
import paper_2310_04610_b200 as E
from paper_2310_04610_b200 import sharded

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
import datetime

dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=60))
E.set_numeric_checks(False)
cfg = (1, 96, 384, 8, 32, "bf16", "check")
full = [t.to(dev) for t in bench.make_inputs(cfg, (0, 96))]
lo, hi = sharded.shard_rows(96, world, rank)
mine = [t[:, lo:hi].contiguous() for t in full[:5]] + [full[5]]
ok = True

# single-GPU reference of the whole problem (every rank computes it alone, no collective)
q, k, v, do, b1, b2 = full
o, lse = E.evoformer_attention_forward(q, k, v, b1, b2)
dq, dk, dv, _, db2 = E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2, deterministic=True)
ref = sharded.ShardedStep(o, lse, dq, dk, dv, None, db2)
for mode in ("blocking", "async"):
    # deterministic backward on both sides: dQ's key-tile partials are summed in a fixed order, so rows
    # can be compared bit for bit
    r = sharded.sharded_fwd_bwd(*mine, async_reduce=(mode == "async"), deterministic=True).wait()
    torch.cuda.synchronize()
    rows_equal = all(torch.equal(getattr(r, n), getattr(ref, n)[:, lo:hi]) for n in ("o", "dq", "dk", "dv"))
    err = ((r.dbias2 - ref.dbias2).abs().max() / ref.dbias2.abs().max()).item()
    print(f"rank {rank} [{mode} NCCL]: rows {lo}..{hi - 1} bit-identical to the 1-GPU run: {rows_equal}; "
          f"dBias2 max rel diff vs 1 GPU {err:.2e}", flush=True)
    ok &= rows_equal and err < 1e-5

# 16-bit dBias2 with the conversion fused into the reduction (fp32 reduce-scatter, per-shard convert,
# bf16 all-gather): equal to the fp32 sum rounded once, up to one bf16 ulp
for mode in ("blocking", "async"):
    r = sharded.sharded_fwd_bwd(*mine, async_reduce=(mode == "async"), dbias_dtype=torch.bfloat16).wait()
    torch.cuda.synchronize()
    want = ref.dbias2.to(torch.bfloat16).float()
    ok16 = r.dbias2.dtype == torch.bfloat16 and bool(
        ((r.dbias2.float() - want).abs() <= want.abs() * 2.0 ** -7 + 1e-30).all())
    print(f"rank {rank} [{mode} bf16 reduce-scatter/convert/all-gather]: within one bf16 ulp of the 1-GPU "
          f"fp32 sum: {ok16}", flush=True)
    ok &= ok16

# in-kernel multicast (NVLS) reduction vs NCCL
os.environ["EVO_MULTICAST"] = "1"
sharded._MC_ENABLED = True
mc = sharded._multicast_dbias2(full[5], None)
if mc is not None:
    r = sharded.sharded_fwd_bwd(*mine)
    torch.cuda.synchronize()
    err = ((r.dbias2 - ref.dbias2).abs().max() / ref.dbias2.abs().max()).item()
    print(f"rank {rank} [multicast NVLS]: dBias2 max rel diff vs 1 GPU {err:.2e}", flush=True)
    ok &= err < 1e-5
else:
    print(f"rank {rank}: symmetric-memory multicast unavailable, NVLS path skipped", flush=True)
dist.barrier()
dist.destroy_process_group()
print(f"rank {rank}: {'PASS' if ok else 'FAIL'}", flush=True)
sys.exit(0 if ok else 1)
