"""Evoformer attention operators over the C-ABI (torch tensors as device memory).

Mirrors the reference operator API for the hot path:
  evoformer_attention_forward   <- evomem::attn_forward_tiled   (attention_tiled.hpp:85-86)
  evoformer_attention_backward  <- evomem::attn_backward_tiled  (attention_tiled.hpp:94-97)
and DeepSpeed's DS4Sci_EvoformerAttention(Q, K, V, [bias1, bias2]) entry point
that OpenFold calls (5-D [Bo, N, L, H, D] tensors, mask bias [Bo, N, 1, 1, L],
pair bias [Bo, 1, H, L, L], scale 1/sqrt(D)).
"""
from __future__ import annotations

import math
from typing import Optional, Sequence, Tuple

import torch

from . import _native as N

_DT = {torch.float32: N.EVO_F32, torch.bfloat16: N.EVO_BF16, torch.float16: N.EVO_F16}
_PATHS = {"auto": N.EVO_PATH_AUTO, "simt": N.EVO_PATH_SIMT, "tcgen05": N.EVO_PATH_TCGEN05}

# NumericError contract of the reference (attention_tiled.cpp:49-65, 125-127, 209): on by default —
# the kernels flag NaN inputs / non-finite logit rows and each call waits for its stream to report
# them. Off, the calls are fully asynchronous (what a training loop that trusts its inputs wants).
_NUMERIC_CHECKS = True


def set_numeric_checks(on: bool) -> bool:
    """Default of `check_numerics` for every operator call; returns the previous setting."""
    global _NUMERIC_CHECKS
    prev, _NUMERIC_CHECKS = _NUMERIC_CHECKS, bool(on)
    return prev


def numeric_checks() -> bool:
    return _NUMERIC_CHECKS


def _as5d(x: torch.Tensor) -> torch.Tensor:
    if x.dim() == 4:
        return x.unsqueeze(0)
    if x.dim() != 5:
        raise N.ValidationError(f"attention tensors must be [Bo, N, L, H, D] or [B, L, H, D], got {tuple(x.shape)}")
    return x


def make_desc(q: torch.Tensor, bias1, bias2, scale: Optional[float], path: str = "auto",
              dbias_dtype: Optional[torch.dtype] = None, check_numerics: Optional[bool] = None,
              deterministic: bool = False) -> N.Desc:
    q5 = _as5d(q)
    Bo, Nr, L, H, D = q5.shape
    if q.dtype not in _DT:
        raise N.ValidationError(f"unsupported dtype {q.dtype}")
    s = 1.0 / math.sqrt(D) if scale is None else float(scale)
    dbt = _DT[dbias_dtype] if dbias_dtype is not None else N.EVO_F32
    d = N.Desc(Bo, Nr, L, H, D, _DT[q.dtype], s, int(bias1 is not None), int(bias2 is not None),
               dbt, _PATHS[path])
    d.check_numerics = int(_NUMERIC_CHECKS if check_numerics is None else check_numerics)
    d.deterministic = int(deterministic)
    return d


def _check_inputs(q, k, v, bias1, bias2):
    q5 = _as5d(q)
    Bo, Nr, L, H, D = q5.shape
    for name, t in (("k", k), ("v", v)):
        if t.shape != q.shape or t.dtype != q.dtype:
            raise N.ValidationError(f"Q, K, V must share one shape and dtype; {name} is {tuple(t.shape)} {t.dtype}")
    if bias1 is not None:
        if tuple(bias1.shape) not in ((Bo, Nr, 1, 1, L),) or bias1.dtype != q.dtype:
            raise N.ValidationError(f"bias1 must be [Bo, N, 1, 1, L] = {(Bo, Nr, 1, 1, L)} of {q.dtype}, got {tuple(bias1.shape)} {bias1.dtype}")
    if bias2 is not None:
        if tuple(bias2.shape) != (Bo, 1, H, L, L) or bias2.dtype != q.dtype:
            raise N.ValidationError(f"bias2 must be [Bo, 1, H, L, L] = {(Bo, 1, H, L, L)} of {q.dtype}, got {tuple(bias2.shape)} {bias2.dtype}")
    for t in (q, k, v, bias1, bias2):
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise N.ValidationError("inputs must be contiguous CUDA tensors")


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def evoformer_attention_forward(q, k, v, bias1=None, bias2=None, scale=None, path: str = "auto",
                                check_numerics: Optional[bool] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """O = softmax(scale*QK^T + bias1 + bias2) V and LSE [B, H, L] (fp32, natural log).
    NumericError on NaN inputs / non-finite logit rows when numeric checks are on."""
    lib = N.load()
    _check_inputs(q, k, v, bias1, bias2)
    d = make_desc(q, bias1, bias2, scale, path, check_numerics=check_numerics)
    o = torch.empty_like(q)
    lse = torch.empty((d.Bo * d.N, d.H, d.L), device=q.device, dtype=torch.float32)
    wsb = lib.evo_attn_fwd_workspace_size(d)
    ws = torch.empty(max(wsb, 1), device=q.device, dtype=torch.uint8)
    N.check(lib.evo_attn_fwd(d, _ptr(q), _ptr(k), _ptr(v), _ptr(bias1), _ptr(bias2), _ptr(o),
                             _ptr(lse), _ptr(ws), wsb, _stream()))
    return o, lse


def evoformer_attention_backward(dout, q, k, v, o, lse, bias1=None, bias2=None, scale=None,
                                 need_dbias1: bool = False, need_dbias2: bool = True,
                                 dbias_dtype: Optional[torch.dtype] = torch.float32,
                                 path: str = "auto", dbias_out: Optional[Tuple] = None,
                                 dbias2_multicast: int = 0, deterministic: bool = False,
                                 check_numerics: Optional[bool] = None):
    """dQ, dK, dV and the broadcast-reduced bias gradients.

    dbias2 is sum over the N (row) axis of dS, reduced inside the kernels, in
    dbias_dtype (float32 = the reference's UpcastF32 policy). dbias_out lets a
    caller pass fp32 accumulators (dbias1, dbias2) that are ADDED to.
    deterministic = AccumPolicy::deterministic (attention_tiled.hpp:35-44): every cross-CTA
    reduction runs in a fixed order, two runs are bit-identical.
    """
    lib = N.load()
    _check_inputs(q, k, v, bias1, bias2)
    if dout.shape != q.shape or o.shape != q.shape or dout.dtype != q.dtype or o.dtype != q.dtype:
        raise N.ValidationError("output and grad_output must match Q/K/V shape and dtype")
    d = make_desc(q, bias1, bias2, scale, path, dbias_dtype, check_numerics, deterministic)
    d.dbias2_multicast = dbias2_multicast or None  # NVSwitch multicast address of a symmetric dBias2 buffer
    if tuple(lse.shape) != (d.Bo * d.N, d.H, d.L) or lse.dtype != torch.float32:
        raise N.ValidationError(f"lse must be [B, H, L] float32, got {tuple(lse.shape)} {lse.dtype}")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    accumulate = dbias_out is not None
    db1 = db2 = None
    if accumulate:
        db1, db2 = dbias_out
    else:
        odt = dbias_dtype if dbias_dtype is not None else torch.float32
        if need_dbias1 and bias1 is not None:
            db1 = torch.empty(bias1.shape, device=q.device, dtype=odt)
        if need_dbias2 and bias2 is not None:
            db2 = torch.empty(bias2.shape, device=q.device, dtype=odt)
    d.need_dbias1 = int(db1 is not None)  # sizes the workspace for the dBias1 path only when asked
    wsb = lib.evo_attn_bwd_workspace_size(d)
    ws = torch.empty(max(wsb, 1), device=q.device, dtype=torch.uint8)
    N.check(lib.evo_attn_bwd(d, _ptr(dout.contiguous()), _ptr(q), _ptr(k), _ptr(v), _ptr(bias1),
                             _ptr(bias2), _ptr(o), _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv),
                             _ptr(db1), _ptr(db2), int(accumulate), _ptr(ws), wsb, _stream()))
    return dq, dk, dv, db1, db2


def evoformer_attention_forward_gated(q, k, v, gate, bias1=None, bias2=None, scale=None, path: str = "auto",
                                      check_numerics: Optional[bool] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """OpenFold-gated attention in one call: o = sigmoid(gate) * attention, the gate
    applied in the forward kernel's epilogue. gate has the shape and dtype of q. Returns (o, lse)."""
    lib = N.load()
    _check_inputs(q, k, v, bias1, bias2)
    if gate.shape != q.shape or gate.dtype != q.dtype or not gate.is_cuda or not gate.is_contiguous():
        raise N.ValidationError("gate must be a contiguous CUDA tensor of the shape and dtype of Q")
    d = make_desc(q, bias1, bias2, scale, path, check_numerics=check_numerics)
    d.has_gate = 1
    o = torch.empty_like(q)
    lse = torch.empty((d.Bo * d.N, d.H, d.L), device=q.device, dtype=torch.float32)
    wsb = lib.evo_attn_fwd_workspace_size(d)
    ws = torch.empty(max(wsb, 1), device=q.device, dtype=torch.uint8)
    N.check(lib.evo_attn_fwd_gated(d, _ptr(q), _ptr(k), _ptr(v), _ptr(bias1), _ptr(bias2), _ptr(gate), _ptr(o),
                                   _ptr(lse), _ptr(ws), wsb, _stream()))
    return o, lse


def evoformer_attention_backward_gated(dout, q, k, v, gate, o, lse, bias1=None, bias2=None, scale=None,
                                       need_dbias1: bool = False, need_dbias2: bool = True,
                                       dbias_dtype: Optional[torch.dtype] = torch.float32, path: str = "auto",
                                       deterministic: bool = False, check_numerics: Optional[bool] = None):
    """Backward of evoformer_attention_forward_gated: dout and o are the GATED output's gradient and
    value. Returns (dq, dk, dv, dgate, dbias1, dbias2); the gate backward is fused into the backward
    preamble's pass over dout and o."""
    lib = N.load()
    _check_inputs(q, k, v, bias1, bias2)
    for name, t in (("dout", dout), ("o", o), ("gate", gate)):
        if t.shape != q.shape or t.dtype != q.dtype or not t.is_contiguous():
            raise N.ValidationError(f"{name} must be contiguous with the shape and dtype of Q")
    d = make_desc(q, bias1, bias2, scale, path, dbias_dtype, check_numerics, deterministic)
    d.has_gate = 1
    if tuple(lse.shape) != (d.Bo * d.N, d.H, d.L) or lse.dtype != torch.float32:
        raise N.ValidationError(f"lse must be [B, H, L] float32, got {tuple(lse.shape)} {lse.dtype}")
    dq, dk, dv, dg = (torch.empty_like(q) for _ in range(4))
    odt = dbias_dtype if dbias_dtype is not None else torch.float32
    db1 = torch.empty(bias1.shape, device=q.device, dtype=odt) if need_dbias1 and bias1 is not None else None
    db2 = torch.empty(bias2.shape, device=q.device, dtype=odt) if need_dbias2 and bias2 is not None else None
    d.need_dbias1 = int(db1 is not None)
    wsb = lib.evo_attn_bwd_workspace_size(d)
    ws = torch.empty(max(wsb, 1), device=q.device, dtype=torch.uint8)
    N.check(lib.evo_attn_bwd_gated(d, _ptr(dout), _ptr(q), _ptr(k), _ptr(v), _ptr(bias1), _ptr(bias2), _ptr(gate),
                                   _ptr(o), _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(dg), _ptr(db1), _ptr(db2),
                                   0, _ptr(ws), wsb, _stream()))
    return dq, dk, dv, dg, db1, db2


def last_launch_count() -> int:
    return int(N.load().evo_attn_last_launch_count())


def resolved_path(q, bias1=None, bias2=None, path="auto", direction: str = "fwd") -> str:
    """Kernel family a call resolves to: direction "fwd" or "bwd" (the tcgen05 backward's envelope is
    narrower: 16-bit, D 16/32, L % 8 == 0)."""
    d = make_desc(q, bias1, bias2, None, path)
    lib = N.load()
    r = (lib.evo_attn_resolved_path if direction == "fwd" else lib.evo_attn_resolved_bwd_path)(d)
    return {N.EVO_PATH_SIMT: "simt", N.EVO_PATH_TCGEN05: "tcgen05"}.get(r, "invalid")


class EvoformerAttentionFunction(torch.autograd.Function):
    """Autograd wrapper: forward saves (q, k, v, o, lse[, gate]) — O(L) extra memory. With a gate the
    saved o is the gated output (the backward needs nothing else, see evo_attn_bwd_gated)."""

    @staticmethod
    def forward(ctx, q, k, v, bias1, bias2, gate=None):
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        b1 = bias1.contiguous() if bias1 is not None else None
        b2 = bias2.contiguous() if bias2 is not None else None
        g = gate.contiguous() if gate is not None else None
        if g is None:
            o, lse = evoformer_attention_forward(q, k, v, b1, b2)
        else:
            o, lse = evoformer_attention_forward_gated(q, k, v, g, b1, b2)
        ctx.save_for_backward(q, k, v, o, lse, b1, b2, g)
        return o

    @staticmethod
    def backward(ctx, grad_o):
        q, k, v, o, lse, b1, b2, g = ctx.saved_tensors
        need1 = b1 is not None and ctx.needs_input_grad[3]
        need2 = b2 is not None and ctx.needs_input_grad[4]
        if g is None:
            dq, dk, dv, db1, db2 = evoformer_attention_backward(
                grad_o.contiguous(), q, k, v, o, lse, b1, b2, need_dbias1=need1, need_dbias2=need2,
                dbias_dtype=q.dtype)
            return dq, dk, dv, db1, db2, None
        dq, dk, dv, dg, db1, db2 = evoformer_attention_backward_gated(
            grad_o.contiguous(), q, k, v, g, o, lse, b1, b2, need_dbias1=need1, need_dbias2=need2,
            dbias_dtype=q.dtype)
        return dq, dk, dv, db1, db2, dg


def DS4Sci_EvoformerAttention(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor,
                              biases: Sequence[Optional[torch.Tensor]], gate: Optional[torch.Tensor] = None
                              ) -> torch.Tensor:
    """DeepSpeed-compatible entry point: Q/K/V [Bo, N, L, H, D]; biases = [mask [Bo, N, 1, 1, L],
    pair [Bo, 1, H, L, L]] (either may be None or omitted). gate (optional, [Bo, N, L, H, D] logits):
    OpenFold's sigmoid output gate fused into the kernels — returns sigmoid(gate) * attention."""
    biases = list(biases)
    if len(biases) > 2:
        raise N.ValidationError("at most two biases (mask, pair)")
    while len(biases) < 2:
        biases.append(None)
    return EvoformerAttentionFunction.apply(Q, K, V, biases[0], biases[1], gate)
