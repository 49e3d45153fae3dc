"""Row-sharding launcher on CPU: world_size-2 gloo process group.

Each rank runs the launcher's own control flow (`sharded_fwd_bwd`) on its contiguous row shard
with oracle-backed operators standing in for the CUDA kernels; the launcher all-reduces the fp32
dBias2 partials over gloo exactly as it does over NCCL on the GPU box. Checks: rows are
independent (O/LSE/dQ/dK/dV of a shard equal the full-problem rows bit for bit) and the
all-reduced dBias2 equals the full-problem dBias2 up to fp32 summation order.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_04610_b200.sharded import reduce_partials_cpu, shard_rows, sharded_fwd_bwd
from tests.util import make_inputs, oracle_fwd_bwd


def test_shard_rows_partition():
    for n in (1, 7, 128, 512, 2048):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_rows(4, 2, 2)


def _oracle_ops():
    """(forward, backward) with the operator signatures of evoformer_attention_*, computed by the
    CPU oracle in float64 (test infrastructure only)."""
    cache = {}

    def fwd(q, k, v, b1, b2):
        res = oracle_fwd_bwd(*(None if t is None else t.numpy() for t in (q, k, v, torch.zeros_like(q), b1, b2)))
        cache["fwd_in"] = (q, k, v, b1, b2)
        return torch.from_numpy(res[0]), torch.from_numpy(res[1])

    def bwd(dout, q, k, v, o, lse, b1, b2, need_dbias1=False, need_dbias2=True, dbias_dtype=torch.float32):
        res = oracle_fwd_bwd(*(None if t is None else t.numpy() for t in (q, k, v, dout, b1, b2)),
                             need_dbias1=need_dbias1)
        dq, dk, dv, db1, db2 = (None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(torch.float32)
                                for a in res[2:])
        return dq, dk, dv, db1 if need_dbias1 else None, db2 if need_dbias2 else None

    return fwd, bwd


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


SHAPE = (1, 6, 40, 2, 8)  # Bo, N, L, H, D


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Bo, Nr, L, H, D = SHAPE
        q, k, v, do, b1, b2 = (None if a is None else torch.from_numpy(a)
                               for a in make_inputs(*SHAPE, dtype="f32", seed=11))
        lo, hi = shard_rows(Nr, world, rank)
        sl = lambda t: t[:, lo:hi].contiguous()
        step = sharded_fwd_bwd(sl(q), sl(k), sl(v), sl(do), sl(b1), b2, ops=_oracle_ops())
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), lo=lo, hi=hi, o=step.o.numpy(), lse=step.lse.numpy(),
                 dq=step.dq.numpy(), dk=step.dk.numpy(), dv=step.dv.numpy(), db2=step.dbias2.numpy())
        # the host-side reduction helper agrees with the launcher's in-place all-reduce
        part = oracle_fwd_bwd(*(t.numpy() for t in (sl(q), sl(k), sl(v), sl(do), sl(b1), b2)))[6]
        red = reduce_partials_cpu(torch.from_numpy(np.ascontiguousarray(part)).to(torch.float32))
        np.save(os.path.join(out_dir, f"red{rank}.npy"), red.numpy())
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_match_full_problem(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    q, k, v, do, b1, b2 = make_inputs(*SHAPE, dtype="f32", seed=11)
    o, lse, dq, dk, dv, _, db2 = oracle_fwd_bwd(q, k, v, do, b1, b2)
    for rank in range(world):
        r = np.load(tmp_path / f"rank{rank}.npz")
        lo, hi = int(r["lo"]), int(r["hi"])
        np.testing.assert_array_equal(r["o"], o[:, lo:hi])
        np.testing.assert_array_equal(r["lse"], lse[lo:hi])  # (B, H, L) with Bo = 1
        np.testing.assert_array_equal(r["dq"], dq[:, lo:hi].astype(np.float32))
        np.testing.assert_array_equal(r["dk"], dk[:, lo:hi].astype(np.float32))
        np.testing.assert_array_equal(r["dv"], dv[:, lo:hi].astype(np.float32))
        # all-reduced fp32 partials == full dBias2 up to fp32 summation order
        scale = np.abs(db2).max()
        assert np.abs(r["db2"] - db2).max() / scale < 1e-6
        assert np.abs(np.load(tmp_path / f"red{rank}.npy") - db2).max() / scale < 1e-6
    r0, r1 = np.load(tmp_path / "rank0.npz"), np.load(tmp_path / "rank1.npz")
    np.testing.assert_array_equal(r0["db2"], r1["db2"])  # every rank holds the same reduced gradient


def _worker_bf16(rank, world, port, out_dir, async_op):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Bo, Nr, L, H, D = SHAPE
        q, k, v, do, b1, b2 = (None if a is None else torch.from_numpy(a)
                               for a in make_inputs(*SHAPE, dtype="f32", seed=11))
        lo, hi = shard_rows(Nr, world, rank)
        sl = lambda t: t[:, lo:hi].contiguous()
        step = sharded_fwd_bwd(sl(q), sl(k), sl(v), sl(do), sl(b1), b2, ops=_oracle_ops(),
                               dbias_dtype=torch.bfloat16, async_reduce=async_op).wait()
        assert step.dbias2.dtype == torch.bfloat16 and step.dbias2.shape == b2.shape
        np.save(os.path.join(out_dir, f"db2_{rank}.npy"), step.dbias2.float().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,async_op", [(2, False), (3, True)])
def test_gloo_bf16_dbias_fused_into_the_reduction(tmp_path, world, async_op):
    """16-bit dBias2 (§8(f)3): fp32 reduce-scatter, per-shard conversion, 16-bit all-gather. Every
    rank holds the same bf16 gradient, equal to the fp32 full-problem sum rounded once (up to one
    bf16 ulp where the fp32 summation order moves a value across a rounding boundary); world 3
    exercises the padded last shard (H*L*L = 3200 is not a multiple of 3)."""
    mp.start_processes(_worker_bf16, args=(world, _free_port(), str(tmp_path), async_op), nprocs=world,
                       join=True, start_method="spawn")
    q, k, v, do, b1, b2 = make_inputs(*SHAPE, dtype="f32", seed=11)
    db2 = oracle_fwd_bwd(q, k, v, do, b1, b2)[6]
    want = torch.from_numpy(np.ascontiguousarray(db2)).to(torch.float32).to(torch.bfloat16).float().numpy()
    got = [np.load(tmp_path / f"db2_{r}.npy") for r in range(world)]
    for g in got[1:]:
        np.testing.assert_array_equal(g, got[0])
    ulp = np.abs(want) * 2.0 ** -7 + 1e-30
    assert np.all(np.abs(got[0] - want) <= ulp)
