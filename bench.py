#!/usr/bin/env python
"""bench.py — EvoformerAttention fwd+bwd TFLOP/s & peak memory on B200 (BASELINE.json metric).

One step = forward + backward of DS4Sci_EvoformerAttention over the whole
workload (all rows, all heads) with mask bias1 and pair bias2, dBias2 reduced
over rows (in-kernel, then NCCL all-reduce across ranks when N > 1).
Default workload: configs[3] of BASELINE.json — OpenFold finetune MSA row
attention N_seq=512 N_res=384 H=8 D=32 bf16 — the configuration the north-star
target (>=50% of dense bf16 peak on 1 B200) is quoted on. --config c1..c5
selects the others. Multi-GPU (--scaling strong, the default): the config's rows
(the MSA-row / triangle-start axis) are split over the ranks and the ranks exchange
only the fp32 dBias2 partial (NCCL all-reduce); --scaling weak gives every rank a
full config's rows.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (Bo, N, L, H, D, dtype, description)
    "c1": (1, 32, 64, 8, 32, "f32", "MSA row attention mask+pair bias fp32, N_seq=32 N_res=64 H=8 D=32"),
    "c2": (1, 128, 256, 8, 32, "bf16", "OpenFold initial-training MSA row attention bf16, N_seq=128 N_res=256 H=8 D=32"),
    "c3": (1, 384, 384, 4, 32, "bf16", "Triangle attention bf16, N_res=384 H=4 D=32, mask+pair bias"),
    "c4": (1, 512, 384, 8, 32, "bf16", "OpenFold finetune MSA row attention bf16, N_seq=512 N_res=384 H=8 D=32"),
    "c5": (1, 2048, 2048, 4, 32, "bf16", "Long-protein triangle attention bf16, N_res=2048 H=4 D=32"),
}
METRIC = "EvoformerAttention fwd+bwd TFLOP/s & peak mem, OpenFold shapes, 1-8 B200"
UNIT = "TFLOP/s"


def flops(B, L, H, D):
    """FlashAttention convention 14*B*H*L^2*D per fwd+bwd: fwd 4, bwd 10."""
    return 14.0 * B * H * L * L * D


def ideal_bytes(B, L, H, D, elem=2):
    """SURVEY §8d byte convention: 24N (bf16 I/O) + 16BHL (LSE, delta) + 16HL^2 (bias2, dbias2) + 4BL."""
    n = B * L * H * D
    return (12 * elem) * n + 16 * B * H * L + 16 * H * L * L + 4 * B * L


def peaks():
    p = {"hbm_gbs": 6534.5, "bf16_tflops": 1667.1, "bf16_tflops_sustained": 1376.6, "source": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "measured"
    except Exception:
        pass
    return p


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, p in zip(names, parts[2:]):
                if p.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [x for x in sm if x > 0.5 * (mx or 1)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_inputs(cfg, rows, pin=False):
    """Synthetic OpenFold-shaped inputs, drawn exactly like the reference's instance generator
    (SeededRng / derived_rng / random_uniform, run.cpp:178-195 — ported in
    paper_2310_04610_b200/inputs.py and pinned bit-for-bit to oracle/_ref): U[-1,1) rounded once to
    the compute dtype, Q, K, V, pair bias from stream 0, dO from stream 2^20, the DS4Sci mask bias1 in
    {0, -1e9} at 10 % from stream 2^21 (key 0 never masked). `rows` = (lo, hi) of the config's rows:
    every rank, the GPU arm and the reference arm draw the same values for the same rows. Host
    tensors."""
    from paper_2310_04610_b200.inputs import random_problem

    Bo, Nr, L, H, D, dt, _ = cfg
    return list(random_problem(Bo, Nr, L, H, D, dtype=dt, seed=7, rows=rows, pin=pin))


def algorithmic(B, L, H, D, elem=2):
    """Per-call algorithmic FLOP and bytes (SURVEY §8(d) conventions) of the forward and backward."""
    n = B * L * H * D
    fwd = {"flop": 4.0 * B * H * L * L * D,
           "bytes": 4 * elem * n + 4 * B * H * L + elem * H * L * L + elem * B * L}  # Q K V in, O + LSE out
    bwd = {"flop": 10.0 * B * H * L * L * D,  # Q K V O dO in, dQ dK dV out, LSE in, bias2 in, dBias2 fp32 out
           "bytes": 8 * elem * n + 4 * B * H * L + elem * H * L * L + 4 * H * L * L + elem * B * L}
    return fwd, bwd


def cpu_baseline(cfg, sample_rows, threads, inputs=None):
    """Reference attn_forward_tiled + attn_backward_tiled (oracle/_ref, the reference's own
    sources) in F32 on the first `sample_rows` rows of the config's inputs (the same values the GPU
    arm computes on), row-sharded over `threads` host threads. Falls back to the C restatement if
    _ref is absent."""
    import numpy as np

    from oracle import oracle as O

    Bo, Nr, L, H, D, dt, _ = cfg
    q, k, v, do, b1, b2 = inputs if inputs is not None else make_inputs(cfg, (0, sample_rows))
    f = lambda t: t[0, :sample_rows].float().numpy().reshape(-1, L, H, D)
    qn, kn, vn, don = (f(t) for t in (q, k, v, do))
    b2n = b2[0, 0].float().numpy()
    t0 = time.perf_counter()
    if O.ref_available():
        O.ref_threaded_f32(qn, kn, vn, b2n, don, threads)
        kind = "reference"
    else:
        p = O.Problem(sample_rows, L, H, D)
        O.fwd_bwd_threaded(p, threads, qn, kn, vn, don, b1[0, :sample_rows].float().numpy().reshape(-1, L), b2n)
        kind = "port"
    dt_s = time.perf_counter() - t0
    tf = flops(sample_rows, L, H, D) / dt_s / 1e12
    return {"value": tf, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"rows 0..{sample_rows - 1} of {Bo * Nr} of {cfg[6]} (the GPU arm's input values), "
                      f"F32 tiled fwd+bwd (tile 64,64,1), {dt_s:.2f} s; mask bias omitted (the reference has no "
                      f"bias1)" if kind == "reference" else f"{sample_rows} rows, oracle port, {dt_s:.2f} s"}


def parity_block(cfg, host, outs, rows, threads):
    """Row sample of this run's own outputs against the oracle (the F32 restatement of
    attention_tiled.cpp:57-340 with the mask term) on the same input values; dBias2 on the reduced
    problem of the sampled rows, computed identically on both sides. Normalized max-abs error
     with the reference-style floored max relative error beside it."""
    import numpy as np

    from oracle import oracle as O

    Bo, Nr, L, H, D, dt, _ = cfg
    q, k, v, do, b1, b2 = host
    f = lambda t: np.ascontiguousarray(t[0, rows].float().numpy(), dtype=np.float64)
    p = O.Problem(len(rows), L, H, D, fmt=O.F32)
    wo, wl, wdq, wdk, wdv, wdb2 = O.fwd_bwd_threaded(
        p, threads, f(q).reshape(-1, L, H, D), f(k).reshape(-1, L, H, D), f(v).reshape(-1, L, H, D),
        f(do).reshape(-1, L, H, D), f(b1).reshape(-1, L), b2[0, 0].double().numpy())
    want = {"O": wo, "LSE": wl.transpose(1, 0, 2), "dQ": wdq, "dK": wdk, "dV": wdv, "dBias2(sample rows)": wdb2}

    def err(g, w):
        g, w = np.asarray(g, np.float64), np.asarray(w, np.float64)
        nmax = float(np.abs(g - w).max() / max(np.abs(w).max(), 1e-30))
        den = np.maximum(np.maximum(np.abs(g), np.abs(w)), max(1e-3 * np.abs(w).max(), 1e-8))
        return {"nmax": nmax, "ref_rel": float((np.abs(g - w) / den).max())}

    res = {n: err(outs[n], want[n]) for n in want}
    tol = 1e-2 if dt != "f32" else 1e-4
    return {"rows": rows, "metric": "normalized max-abs error vs the oracle on identical inputs",
            "tol": tol, "pass": all(r["nmax"] <= tol for r in res.values()), "errors": res}


def run_reference_arm(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    Bo, Nr, L, H, D, dt, desc = cfg
    # bounded sample per step: one row per host thread, shrunk so that the whole (warmup + steps)
    # run stays within ~4 minutes; the rows' values are the GPU arm's (same generator, same streams)
    sample = min(Bo * Nr, threads)
    host = make_inputs(cfg, (0, sample))
    first = cpu_baseline(cfg, sample, threads, host)
    per_step = flops(sample, L, H, D) / (first["value"] * 1e12)
    budget = 240.0 / max(1, args.steps + args.warmup)
    if per_step > budget:
        sample = max(1, int(sample * budget / per_step))
        threads = min(threads, sample)
    for _ in range(args.warmup - 1):
        cpu_baseline(cfg, sample, threads, host)
    vals = [cpu_baseline(cfg, sample, threads, host) for _ in range(args.steps)]
    v = statistics.median(x["value"] for x in vals)
    ms = flops(sample, L, H, D) / (v * 1e12) * 1e3
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference SeededRng streams)",
            "config": {"workload": desc, "config": args.config, "Bo": Bo, "N": Nr, "L": L, "H": H, "D": D,
                       "parallelism": f"cpu_threads{threads}"},
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": vals[0]["kind"],
                             "sample": vals[0]["sample"]},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


_JSON_FD = 1


def emit(line: dict):
    os.write(_JSON_FD, (json.dumps(line) + "\n").encode())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--e2e-streams", type=int, default=1,
                    help="copy streams per direction in the end-to-end run (copy engines share the PCIe link)")
    ap.add_argument("--e2e-steps", type=int, default=20,
                    help="end-to-end steps timed (pipeline fill and drain amortised over them)")
    ap.add_argument("--all-configs", action="store_true", help="also time c1..c5 and attach them")
    ap.add_argument("--reduce", default="async", choices=["blocking", "async"],
                    help="multi-GPU dBias2 all-reduce: blocking (after the backward, on the compute stream) or "
                         "async (NCCL's stream, overlapping the next step's forward)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong: the config's rows split over ranks (headline); weak: each rank owns a "
                         "full config's rows")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    # stdout carries exactly one JSON line: anything else written to fd 1 (library banners such as
    # NCCL's version line) is sent to stderr, the JSON goes to the saved original stdout.
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_2310_04610_b200 as E
    from paper_2310_04610_b200.sharded import shard_rows, sharded_fwd_bwd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import datetime

        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=120))
    # Timed loops run asynchronously: the NumericError host round trip (a stream sync per call) is
    # off there; the checked mode is timed separately below and reported beside the headline.
    E.set_numeric_checks(False)

    Bo, Nr, L, H, D, dt, desc = cfg

    def rows_of(r, n):
        return shard_rows(Nr, n, r) if args.scaling == "strong" else (0, Nr)

    lo, hi = rows_of(rank, world)
    host = make_inputs(cfg, (lo, hi), pin=True)
    q, k, v, do, b1, b2 = (t.to(dev) for t in host)
    B_local = Bo * (hi - lo)
    B_total = Bo * Nr if args.scaling == "strong" else Bo * Nr * world

    pending = []

    def step():
        # multi-GPU: the dBias2 all-reduce of this step runs asynchronously (NCCL's stream) and overlaps
        # the next step's forward; the previous step's reduction is waited for here, the last one before
        # the closing event
        async_reduce = world > 1 and args.reduce == "async"
        r = sharded_fwd_bwd(q, k, v, do, b1, b2, async_reduce=async_reduce)
        while pending:
            pending.pop().wait()
        if async_reduce:
            pending.append(r)
        return r

    def drain():
        while pending:
            pending.pop().wait()

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- warm-up + launch count
    for _ in range(args.warmup):
        step()
    drain()
    torch.cuda.synchronize()
    E.evoformer_attention_forward(q, k, v, b1, b2)
    n_fwd = E.last_launch_count()
    o, lse = E.evoformer_attention_forward(q, k, v, b1, b2)
    E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2, need_dbias1=False)
    n_bwd = E.last_launch_count()
    path = E.resolved_path(q, b1, b2)
    bwd_path = E.resolved_path(q, b1, b2, direction="bwd")

    # ---- peak memory of one fwd+bwd beyond the I/O tensors
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    r = step()
    drain()
    torch.cuda.synchronize()
    outs = sum(t.numel() * t.element_size() for t in (r.o, r.lse, r.dq, r.dk, r.dv) if t is not None)
    outs += sum(t.numel() * t.element_size() for t in (r.dbias1, r.dbias2) if t is not None)
    peak_extra = torch.cuda.max_memory_allocated() - base - outs
    del r

    # ---- timed region: K steps, barrier + sync on both sides, CUDA events on the launching stream
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        t_host = time.perf_counter()
        for _ in range(args.steps):
            step()
        drain()
        t_host = time.perf_counter() - t_host
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    total_flops = flops(B_total, L, H, D)
    value = total_flops / (ms * 1e-3) / 1e12

    def time_call(fn, n):
        for _ in range(2):  # warm (allocator, first-launch setup)
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(n):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    # the same step with the reference's NumericError checks on (each call waits for its stream)
    E.set_numeric_checks(True)
    barrier()
    ms_checked = time_call(lambda: (step(), drain()), max(5, args.steps // 4))
    E.set_numeric_checks(False)

    # the same step with OpenFold's sigmoid output gate fused: gated forward + backward
    gate = torch.empty_like(q).uniform_(-3, 3)
    og, lse_g = E.evoformer_attention_forward_gated(q, k, v, gate, b1, b2)
    gated_ms = time_call(lambda: (E.evoformer_attention_forward_gated(q, k, v, gate, b1, b2),
                                  E.evoformer_attention_backward_gated(do, q, k, v, gate, og, lse_g, b1, b2)),
                         max(10, args.steps // 4))
    del gate, og, lse_g

    # the pair-bias projection feeding bias2: LayerNorm(z)·W → [Bo, 1, H, L, L] and its
    # backward from dBias2, z = [Bo, L, L, c_z = 128] (OpenFold's pair channels), timed alone
    pair_bias = None
    if b2 is not None and dt != "f32":
        cz = 128
        zp = (torch.randn(Bo, L, L, cz, device=dev) * 2).to(q.dtype)
        lw, lb = torch.ones(cz, device=dev), torch.zeros(cz, device=dev)
        wz = torch.randn(H, cz, device=dev) / cz ** 0.5
        gb = torch.randn(Bo, 1, H, L, L, device=dev)
        pf = time_call(lambda: E.pair_bias_forward(zp, lw, lb, wz), 20)
        pb = time_call(lambda: E.pair_bias_backward(gb, zp, lw, lb, wz), 20)
        zbytes = zp.numel() * zp.element_size()
        pair_bias = {"c_z": cz, "fwd_ms": pf, "bwd_ms": pb,
                     "fwd_gbs": (zbytes + gb.numel() * zp.element_size()) / pf / 1e6,
                     "bwd_gbs": (2 * zbytes + gb.numel() * 4) / pb / 1e6,
                     "what": "LayerNorm(z)·W -> bias2 in the attention's layout, and its backward from fp32 dBias2"}
        del zp, gb

    allreduce_us = None
    if world > 1 and b2 is not None:  # the dBias2 all-reduce alone (fp32, H*L*L), blocking on the stream
        buf = torch.zeros(b2.numel(), device=dev, dtype=torch.float32)
        barrier()
        allreduce_us = 1e3 * time_call(lambda: dist.all_reduce(buf), 20)

    # ---- per-call timing (forward call, backward call) on the launching stream; the dominant call's
    # roofline against the bound of the SURVEY §8(d) model (max of the FLOP and byte times)
    o, lse = E.evoformer_attention_forward(q, k, v, b1, b2)
    nk = max(10, args.steps // 2)
    fwd_ms = time_call(lambda: E.evoformer_attention_forward(q, k, v, b1, b2), nk)
    bwd_ms = time_call(lambda: E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2,
                                                              need_dbias1=False), nk)
    pk = peaks()
    elem = 4 if dt == "f32" else 2
    a_fwd, a_bwd = algorithmic(B_local, L, H, D, elem)
    dom_name, dom, dom_ms = ("bwd", a_bwd, bwd_ms) if bwd_ms >= fwd_ms else ("fwd", a_fwd, fwd_ms)
    t_flop = dom["flop"] / (pk["bf16_tflops"] * 1e12)
    t_hbm = dom["bytes"] / (pk["hbm_gbs"] * 1e9)
    bound = "hbm" if t_hbm >= t_flop else "tensor"
    achieved = dom["bytes"] / (dom_ms * 1e-3) / 1e9 if bound == "hbm" else dom["flop"] / (dom_ms * 1e-3) / 1e12
    peak = pk["hbm_gbs"] if bound == "hbm" else pk["bf16_tflops"]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tj = json.load(f)  # per-call DRAM bytes (the backward call = preamble + main kernel + conversions)
            traffic = tj.get(f"{args.config}_{dom_name}_call_{path}", tj.get(f"{args.config}_{dom_name}_{path}"))
    except Exception:
        pass
    roofline = {"bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": f"{dom_name} call ({path})",
                "peak_source": pk["source"],
                "algorithmic": {"flop": dom["flop"], "bytes": dom["bytes"], "t_flop_us": t_flop * 1e6,
                                "t_hbm_us": t_hbm * 1e6},
                "tensor_frac": dom["flop"] / (dom_ms * 1e-3) / 1e12 / pk["bf16_tflops"],
                "hbm_frac": dom["bytes"] / (dom_ms * 1e-3) / 1e9 / pk["hbm_gbs"],
                "kernels": {"fwd": {"ms": fwd_ms, "tflops": a_fwd["flop"] / fwd_ms / 1e9,
                                    "gbs": a_fwd["bytes"] / fwd_ms / 1e6},
                            "bwd": {"ms": bwd_ms, "tflops": a_bwd["flop"] / bwd_ms / 1e9,
                                    "gbs": a_bwd["bytes"] / bwd_ms / 1e6}},
                "step_roofline_frac": (max(flops(B_local, L, H, D) / (pk["bf16_tflops"] * 1e12),
                                           ideal_bytes(B_local, L, H, D, elem) / (pk["hbm_gbs"] * 1e9))
                                       / (ms * 1e-3))}

    # ---- end to end through the public API with pinned host buffers. Every step copies its inputs
    # host->device and its gradients device->host; the copies of neighbouring steps overlap the
    # compute on separate streams (inputs double-buffered), which is how a training loop feeds it.
    host_in = host
    dev_sets = [[torch.empty_like(t, device=dev) for t in host_in] for _ in range(2)]
    r = step()
    drain()
    host_out = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in (r.dq, r.dk, r.dv, r.dbias2)]
    h2d = sum(t.numel() * t.element_size() for t in host_in)
    d2h = sum(t.numel() * t.element_size() for t in host_out)
    # copies spread over args.e2e_streams streams per direction (several copy engines share PCIe)
    ns = max(1, args.e2e_streams)
    s_ins = [torch.cuda.Stream() for _ in range(ns)]
    s_outs = [torch.cuda.Stream() for _ in range(ns)]
    s_in = s_ins[0]

    def e2e_run(nsteps):
        ready = [[torch.cuda.Event() for _ in range(ns)] for _ in range(2)]
        free = [torch.cuda.Event() for _ in range(2)]
        for f in free:
            f.record(stream)

        def upload(slot):
            for si, sin in enumerate(s_ins):
                with torch.cuda.stream(sin):
                    sin.wait_event(free[slot])
                    for k_, (hs, ds) in enumerate(zip(host_in, dev_sets[slot])):
                        if k_ % ns == si:
                            ds.copy_(hs, non_blocking=True)
                    ready[slot][si].record(sin)

        upload(0)
        for i in range(nsteps):
            cur = i % 2
            if i + 1 < nsteps:
                upload(1 - cur)
            for ev in ready[cur]:
                stream.wait_event(ev)
            rr = sharded_fwd_bwd(*dev_sets[cur]).wait()
            free[cur].record(stream)
            done = torch.cuda.Event()
            done.record(stream)
            for so_i, sout in enumerate(s_outs):
                with torch.cuda.stream(sout):
                    sout.wait_event(done)
                    for k_, (hd, t_) in enumerate(zip(host_out, (rr.dq, rr.dk, rr.dv, rr.dbias2))):
                        if k_ % ns == so_i:
                            t_.record_stream(sout)
                            hd.copy_(t_, non_blocking=True)
        for sout in s_outs:
            stream.wait_stream(sout)

    e2e_run(2)
    torch.cuda.synchronize()
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for sin in s_ins:
        sin.wait_stream(stream)
    e2e_run(args.e2e_steps)
    b.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = a.elapsed_time(b) / args.e2e_steps
    t = torch.tensor([e2e_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    extra = {}
    if args.all_configs and world == 1:
        for name, c in CONFIGS.items():
            if name == args.config:
                continue
            qq, kk, vv, dd, bb1, bb2 = (x.to(dev) for x in make_inputs(c, (0, c[1])))
            for _ in range(3):
                sharded_fwd_bwd(qq, kk, vv, dd, bb1, bb2)
            n = 20 if name != "c5" else 3
            mm = time_call(lambda: sharded_fwd_bwd(qq, kk, vv, dd, bb1, bb2), n)
            extra[name] = {"ms_per_step": mm, "tflops": flops(c[0] * c[1], c[2], c[3], c[4]) / mm / 1e9,
                           "path": E.resolved_path(qq, bb1, bb2)}
            del qq, kk, vv, dd, bb1, bb2
            torch.cuda.empty_cache()
        # C3 as the triangle END-node variant: raw [N_res, N_res, H, D] tensors attended over axis 0,
        # run in place through the variant layer (descriptor axes_swapped; autograd fwd+bwd)
        Lt, Ht, Dt = 384, 4, 32
        g = torch.Generator(device=dev).manual_seed(7)
        rr = lambda *sh: (torch.rand(*sh, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
        tq, tk, tv = (rr(Lt, Lt, Ht, Dt).requires_grad_(True) for _ in range(3))
        tb, tdo = rr(Ht, Lt, Lt).requires_grad_(True), rr(Lt, Lt, Ht, Dt)
        tm = torch.zeros(Lt, Lt, device=dev, dtype=torch.bfloat16)
        tri = lambda: E.variant_attention("tri_end", tq, tk, tv, tb, tm).backward(tdo)
        for _ in range(3):
            tri()
        mm = time_call(tri, 20)
        extra["c3_tri_end_raw_layout"] = {"ms_per_step": mm, "tflops": flops(Lt, Lt, Ht, Dt) / mm / 1e9,
                                          "path": "tcgen05 (axes_swapped)"}
        del tq, tk, tv, tb, tdo, tm
        torch.cuda.empty_cache()

    th = os.cpu_count() or 1
    parity = None
    if rank == 0 and not args.no_parity:
        # this run's own outputs on a row sample of rank 0's shard, against the oracle on the same values
        try:
            nloc = hi - lo
            rows = sorted(set(int(round(x)) for x in [0, nloc // 3, (2 * nloc) // 3, nloc - 1]))
            if args.config == "c5":
                rows = [0, nloc - 1]
            # rank 0 alone: the operators directly (sharded_fwd_bwd would issue an all-reduce the other
            # ranks never join)
            fo, fl = E.evoformer_attention_forward(q, k, v, b1, b2)
            fdq, fdk, fdv, _, _ = E.evoformer_attention_backward(do, q, k, v, fo, fl, b1, b2, need_dbias1=False)
            idx = torch.tensor(rows, device=dev)
            sel = lambda x: x[0].index_select(0, idx).float().cpu().numpy()
            outs = {"O": sel(fo), "LSE": fl.index_select(0, idx).cpu().numpy(), "dQ": sel(fdq),
                    "dK": sel(fdk), "dV": sel(fdv)}
            sub = lambda x: x[:, idx].contiguous()
            # dBias2 of the reduced problem of the sampled rows, on this rank alone
            so, sl = E.evoformer_attention_forward(sub(q), sub(k), sub(v), sub(b1), b2)
            sdb2 = E.evoformer_attention_backward(sub(do), sub(q), sub(k), sub(v), so, sl, sub(b1), b2)[4]
            outs["dBias2(sample rows)"] = sdb2[0, 0].cpu().numpy()
            parity = parity_block(cfg, host, outs, rows, th)
            parity["rows"] = [lo + x for x in rows]
        except Exception as e:  # reported, never hidden
            parity = {"pass": False, "error": repr(e)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sample = max(th, (Bo * Nr) // 64) if args.config != "c5" else 2
            cpu = cpu_baseline(cfg, min(sample, hi - lo), th, host)
        except Exception as e:  # reported, never silently substituted
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable", "sample": repr(e)}

    if rank == 0:
        naive = 3 * H * B_local * L * L * elem
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": dt, "data": "synthetic (reference SeededRng streams, seed 7)",
            "config": {"workload": desc, "config": args.config, "Bo": Bo, "N": Nr, "L": L, "H": H,
                       "D": D, "biases": "mask bias1 [Bo,N,1,1,L] + pair bias2 [Bo,1,H,L,L]",
                       "rows_per_rank": B_local, "rows_total": B_total,
                       "parallelism": f"rows_sharded_dp{world}", "kernel_path": path, "bwd_kernel_path": bwd_path,
                       "dbias2_allreduce": args.reduce if world > 1 else None,
                       "numeric_checks": "off in the timed loop (ms_per_step_checked: on)",
                       "l2": "inputs+outputs larger than L2 (no flush needed)"
                       if ideal_bytes(B_local, L, H, D, elem) > 126e6 else "working set smaller than L2 (not flushed)"},
            "ms_per_step_checked": ms_checked,
            "host_enqueue_ms_per_step": t_host * 1e3 / args.steps,
            "dbias2_allreduce_us": allreduce_us,
            "gated": {"ms_per_step": gated_ms, "tflops": flops(B_local, L, H, D) / gated_ms / 1e9,
                      "what": "fwd+bwd with the fused sigmoid output gate (this rank's rows, no all-reduce)"},
            "pair_bias": pair_bias,
            "peak_mem": {"extra_bytes_per_rank": int(peak_extra), "naive_logits_bytes": naive,
                         "o_l_plan_bytes": 8 * B_local * H * L + 4 * H * L * L,
                         # the reference attn-bench column (run.cpp:223-234): naive / tiled peak
                         "reduction_ratio": naive / max(int(peak_extra), 1)},
            "roofline": roofline,
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": {"value": total_flops / (e2e_ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": (n_fwd + n_bwd) * args.steps,
            "clocks": clk.summary(),
        }
        if extra:
            line["other_configs"] = extra
        emit(line)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
