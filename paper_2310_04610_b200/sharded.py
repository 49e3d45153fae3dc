"""Row-sharding launcher: one process per GPU, rows of the batch axis split
contiguously over ranks, NCCL all-reduce of the pair-bias gradient only.

Rows (MSA rows / triangle start nodes) are independent for O, LSE, dQ, dK, dV
(attention_tiled.cpp:83-177, 254-330); the only coupling is dBias2 =
sum_b dS (attention_tiled.cpp:318-323), the broadcast-reverse sum. Each rank
reduces its rows inside the kernels into an fp32 partial; the launcher then
all-reduces that partial (sum, fp32) over NVLink. bias1 is per-row, so its
gradient needs no communication.
"""
from __future__ import annotations

import os

from dataclasses import dataclass
from typing import Optional, Tuple

import torch
import torch.distributed as dist

from ._native import UnsupportedError
from .evoformer_attention import evoformer_attention_backward, evoformer_attention_forward


def shard_rows(n_rows: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous near-equal split of [0, n_rows): rank r gets [lo, hi)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    lo = n_rows * rank // world
    hi = n_rows * (rank + 1) // world
    return lo, hi


@dataclass
class ShardedStep:
    o: torch.Tensor
    lse: torch.Tensor
    dq: torch.Tensor
    dk: torch.Tensor
    dv: torch.Tensor
    dbias1: Optional[torch.Tensor]
    dbias2: Optional[torch.Tensor]
    pending: Optional[object] = None  # in-flight dBias2 reduction (async_reduce)

    def wait(self) -> "ShardedStep":
        """Make the current stream wait for the in-flight dBias2 reduction; dbias2 is then final."""
        if self.pending is not None:
            self.pending.wait()
            self.pending = None
        return self


_SIDE = {}


def _side_stream(device):
    if device not in _SIDE:
        _SIDE[device] = torch.cuda.Stream(device)
    return _SIDE[device]


def reduce_dbias2(db2, dbias_dtype=torch.float32, group=None, async_op=False):
    """Sum the ranks' fp32 dBias2 partials; returns (result, pending work or None).

    fp32 result: one fp32 all-reduce. 16-bit result (§8(f)3, the dBias convert fused into the
    all-reduce): reduce-scatter of the fp32 partials, each rank converts its 1/world shard, all-gather
    of the 16-bit shards — no full-size conversion pass, and the gather half moves 16-bit values (3/4
    of the fp32 all-reduce's bytes). The sum is fp32 either way (the reference's UpcastF32 policy,
    attention_tiled.cpp:318-323); only the final value is rounded. async_op: the collectives (and the
    shard conversion, on a side stream) are ordered after the work queued so far and overlap what the
    caller queues next; wait() on the returned work before reading the result.
    """
    if dbias_dtype == torch.float32:
        return db2, dist.all_reduce(db2, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
    world = dist.get_world_size(group)
    n = db2.numel()
    per = -(-n // world)
    flat = db2.reshape(-1)
    if per * world != n:
        flat = torch.cat([flat, flat.new_zeros(per * world - n)])
    shard = flat.new_empty(per)
    out = torch.empty(per * world, dtype=dbias_dtype, device=db2.device)
    res = out[:n].view(db2.shape)
    if async_op and db2.is_cuda:
        rs = dist.reduce_scatter_tensor(shard, flat, op=dist.ReduceOp.SUM, group=group, async_op=True)
        side = _side_stream(db2.device)
        with torch.cuda.stream(side):
            rs.wait()  # the side stream waits for the reduce-scatter (not the compute stream)
            s16 = shard.to(dbias_dtype)
            ag = dist.all_gather_into_tensor(out, s16, group=group, async_op=True)
        for t in (flat, shard, s16, out):
            t.record_stream(side)
        return res, ag
    work = dist.reduce_scatter_tensor(shard, flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
    if work is not None:
        work.wait()
    work = dist.all_gather_into_tensor(out, shard.to(dbias_dtype), group=group, async_op=async_op)
    return res, work


def sharded_fwd_bwd(q, k, v, dout, bias1, bias2, group=None, dbias_dtype: torch.dtype = torch.float32,
                    need_dbias1: bool = False, ops=None, async_reduce: bool = False,
                    deterministic: bool = False) -> ShardedStep:
    """Forward + backward on this rank's row shard, dBias2 all-reduced.

    q/k/v/dout/bias1 are this rank's rows ([Bo, n_local, L, H, D]); bias2 is the full pair bias.
    The kernels reduce this rank's rows of dS into an fp32 dBias2 partial; one fp32 sum
    all-reduce over the group completes it — or, for a 16-bit dbias_dtype, an fp32
    reduce-scatter, the per-shard conversion and a 16-bit all-gather (`reduce_dbias2`). The mask-bias gradient is off by
    default (the MSA mask carries no gradient in OpenFold; the headline step produces dQ, dK, dV
    and dBias2). `ops` = (forward, backward) overrides the CUDA operators (used by the CPU
    gloo tests to drive the same control flow with the oracle). async_reduce: the all-reduce is
    issued without blocking the compute stream (NCCL runs it on its own stream, ordered after this
    backward), so it overlaps whatever the caller launches next (the next layer's or step's
    forward); call .wait() on the result before reading dbias2.
    """
    fwd, bwd = ops if ops is not None else (evoformer_attention_forward, evoformer_attention_backward)
    o, lse = fwd(q, k, v, bias1, bias2)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    need1 = need_dbias1 and bias1 is not None
    mc = _multicast_dbias2(bias2, group) if (world > 1 and ops is None and bias2 is not None) else None
    if mc is not None:
        # in-kernel cross-GPU reduction: the backward's dBias2 strip flush adds through the NVSwitch
        # multicast address into every rank's replica (multimem.red), so no all-reduce is issued
        buf, handle = mc
        buf.zero_()
        handle.barrier(channel=0)  # every replica is zero before any rank adds
        try:
            # dbias_out holds fp32 accumulators the kernels ADD to: the mask-bias gradient (per row,
            # rank-local) needs its own zeroed buffer on this path too
            db1 = torch.zeros(bias1.shape, device=q.device, dtype=torch.float32) if need1 else None
            dq, dk, dv, _, _ = bwd(dout, q, k, v, o, lse, bias1, bias2, need_dbias1=need1,
                                   need_dbias2=True, dbias_dtype=torch.float32, dbias_out=(db1, buf),
                                   dbias2_multicast=handle.multicast_ptr)
            handle.barrier(channel=0)  # every rank's adds have landed in every replica
            db2 = buf.view(bias2.shape).clone()
        except UnsupportedError:  # shape outside the tcgen05 backward: reduce with NCCL instead
            handle.barrier(channel=0)
            mc = None
    if mc is None:
        kw = {"deterministic": True} if deterministic else {}
        dq, dk, dv, db1, db2 = bwd(
            dout, q, k, v, o, lse, bias1, bias2, need_dbias1=need1,
            need_dbias2=bias2 is not None, dbias_dtype=torch.float32, **kw)
        if db2 is not None and world > 1:
            db2, work = reduce_dbias2(db2, dbias_dtype, group, async_op=async_reduce)
            if db1 is not None and dbias_dtype != torch.float32:
                db1 = db1.to(dbias_dtype)
            return ShardedStep(o, lse, dq, dk, dv, db1, db2, pending=work if async_reduce else None)
    if db2 is not None and dbias_dtype != torch.float32:
        db2 = db2.to(dbias_dtype)
    if db1 is not None and dbias_dtype != torch.float32:
        db1 = db1.to(dbias_dtype)
    return ShardedStep(o, lse, dq, dk, dv, db1, db2)


_MC = {}
# Opt-in: measured on B200 x2 at C4 the in-kernel multicast flush (144 CTAs x 96 KB of 16-byte
# multimem.red per GPU, NVLS op-rate bound) adds ~190 us to the backward while NCCL's all-reduce of
# the reduced 4.7 MB costs ~42 us, so the NCCL path is the default.
_MC_ENABLED = os.environ.get("EVO_MULTICAST", "0") == "1"


def _multicast_dbias2(bias2, group):
    """(buffer, handle) of a symmetric fp32 dBias2 buffer with NVSwitch multicast, cached per group and
    shape; None when symmetric memory or multicast is unavailable (the launcher then all-reduces)."""
    if not _MC_ENABLED or not bias2.is_cuda:
        return None
    key = (id(group), tuple(bias2.shape), bias2.device)
    if key in _MC:
        return _MC[key]
    res = None
    try:
        import torch.distributed._symmetric_memory as symm_mem

        idx = bias2.device.index if bias2.device.index is not None else torch.cuda.current_device()
        if symm_mem._SymmetricMemory.has_multicast_support(symm_mem.DeviceType.CUDA, idx):
            buf = symm_mem.empty(bias2.numel(), dtype=torch.float32, device=bias2.device)
            handle = symm_mem.rendezvous(buf, group if group is not None else dist.group.WORLD)
            if handle.multicast_ptr:
                res = (buf, handle)
    except Exception:
        res = None
    _MC[key] = res
    return res


def reduce_partials_cpu(partials, group=None) -> torch.Tensor:
    """Host-side form of the dBias2 reduction used by the gloo tests: sum the
    fp32 partial of every rank (same op the NCCL path issues)."""
    t = partials.clone()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t
