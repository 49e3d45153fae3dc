"""Evoformer attention variants over the fused operator.

Mirrors the reference's variant layer:
  AttentionVariant / variant_name / variant_from_name / variant_has_bias
      <- attention.hpp:12-19, attention.cpp:10-32
  layout_from_msa / inverse_permutation
      <- attention.hpp:65-77, attention.cpp:101-124, 160-166
  problem validation (bias iff variant, (H, L, L) bias, B == L for triangles, finite scale)
      <- attention.cpp:48-88

Raw inputs arrive in the model's own axes: MSA variants as (N_msa, N_res, H, D), triangular as
(N_res, N_res, H, D). Row-wise and start-node attend over axis 1 (canonical as-is); column-wise
and end-node attend over axis 0, so their canonical (B, L, H, D) view swaps axes 0 and 1
(attention.cpp:109-119). The kernels take that layout in place (descriptor `axes_swapped`: the TMA
maps trade the L and B strides; O, dQ, dK, dV are written back in the raw layout), so no transposed
copy is made in either direction and a caller sees the reference's semantics in its own axes. bias is the reference's (H, L, L) pair bias (broadcast over B); mask is the DS4Sci bias1
extension, (B, L) in canonical axes — additive, 0 or a large negative value.

`variant_forward` is the copy-free inference forward: for msa_col / tri_end the kernels read Q/K/V and
write O in the raw layout through the descriptor's `axes_swapped` strides (TMA maps with the L and
B strides traded), so no transposed copy is made.

`chunked_forward` is the inference mode: the forward over row chunks with one output buffer, so
the kernels' per-call working set is bounded by the chunk (rows are independent in the forward).
"""
from __future__ import annotations

import enum
import math
from typing import NamedTuple, Optional, Tuple

import torch

from . import _native as N
from .evoformer_attention import (_DT, _PATHS, _ptr, _stream, EvoformerAttentionFunction,
                                  evoformer_attention_forward, numeric_checks)


class AttentionVariant(enum.Enum):
    """attention.hpp:14 — the four biased-axial-attention variants."""
    MsaRowWise = "msa_row"
    MsaColumnWise = "msa_col"
    TriangularStartNode = "tri_start"
    TriangularEndNode = "tri_end"


def variant_name(v: AttentionVariant) -> str:
    return v.value


def variant_from_name(name: str) -> AttentionVariant:
    """attention.cpp:25-32: unknown names are a ValidationError."""
    for v in AttentionVariant:
        if v.value == name:
            return v
    raise N.ValidationError(f"unknown attention variant '{name}' (expected msa_row|msa_col|tri_start|tri_end)")


def variant_has_bias(v: AttentionVariant) -> bool:
    """attention.hpp:16-18: every variant but column-wise carries a pair bias."""
    return v is not AttentionVariant.MsaColumnWise


_SWAP = (1, 0, 2, 3)
_IDENT = (0, 1, 2, 3)


class CanonicalLayout(NamedTuple):
    """attention.hpp:65-70."""
    tensor: torch.Tensor          # (B, L, H, D), contiguous
    permutation: Tuple[int, int, int, int]
    batch_extent: int
    attended_extent: int


def inverse_permutation(perm) -> Tuple[int, int, int, int]:
    """attention.cpp:160-166."""
    inv = [0, 0, 0, 0]
    for k, a in enumerate(perm):
        inv[a] = k
    return tuple(inv)


def _as_variant(v) -> AttentionVariant:
    return v if isinstance(v, AttentionVariant) else variant_from_name(v)


def layout_from_msa(variant, raw: torch.Tensor) -> CanonicalLayout:
    """attention.cpp:101-124: permute a raw rank-4 tensor into canonical (B, L, H, D)."""
    variant = _as_variant(variant)
    if raw.dim() != 4:
        raise N.ValidationError(f"layout_from_msa expects a rank-4 tensor, got {tuple(raw.shape)}")
    perm = _SWAP if variant in (AttentionVariant.MsaColumnWise, AttentionVariant.TriangularEndNode) else _IDENT
    t = raw.permute(*perm).contiguous()
    return CanonicalLayout(t, perm, int(t.shape[0]), int(t.shape[1]))


def validate_variant_problem(variant, q, k, v, bias=None, mask=None, scale=None) -> None:
    """attention.cpp:48-88 on canonical (B, L, H, D) tensors, plus the mask shape (DS4Sci bias1)."""
    variant = _as_variant(variant)
    if q.dim() != 4:
        raise N.ValidationError(f"attention tensors must be rank-4 (B, L, H, D), got {tuple(q.shape)}")
    if q.shape != k.shape or q.shape != v.shape:
        raise N.ValidationError(f"Q, K, V must share one shape; got {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    if q.dtype != k.dtype or q.dtype != v.dtype:
        raise N.ValidationError("Q, K, V must share one numeric format")
    B, L, H, _ = q.shape
    needs = variant_has_bias(variant)
    if needs != (bias is not None):
        raise N.ValidationError(f"variant {variant.value} " + ("requires a bias tensor" if needs else "does not take a bias"))
    if bias is not None:
        if tuple(bias.shape) != (H, L, L):
            raise N.ValidationError(f"bias must be (H, L, L) = ({H}, {L}, {L}), got {tuple(bias.shape)}")
        if bias.dtype != q.dtype:
            raise N.ValidationError("bias must share the problem numeric format")
    if mask is not None:
        if tuple(mask.shape) != (B, L):
            raise N.ValidationError(f"mask must be (B, L) = ({B}, {L}) in canonical axes, got {tuple(mask.shape)}")
        if mask.dtype != q.dtype:
            raise N.ValidationError("mask must share the problem numeric format")
    if variant in (AttentionVariant.TriangularStartNode, AttentionVariant.TriangularEndNode) and B != L:
        raise N.ValidationError(f"triangular variants require B == L (N_res, N_res), got ({B}, {L})")
    if scale is not None and not math.isfinite(scale):
        raise N.NumericError("attention scale must be finite")


def variant_attention(variant, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                      bias: Optional[torch.Tensor] = None, mask: Optional[torch.Tensor] = None,
                      ) -> torch.Tensor:
    """Biased axial attention of one variant on raw (model-axis) Q/K/V; differentiable in Q, K, V,
    bias and mask. Returns O in the raw axes. Scale is 1/sqrt(D) (attention.cpp:43-45)."""
    variant = _as_variant(variant)
    swap = variant in (AttentionVariant.MsaColumnWise, AttentionVariant.TriangularEndNode)
    perm = _SWAP if swap else _IDENT
    qc, kc, vc = (t.permute(*perm) for t in (q, k, v))
    validate_variant_problem(variant, qc, kc, vc, bias, mask)
    if not all(t.is_cuda for t in (q, k, v, bias, mask) if t is not None):
        raise N.ValidationError("inputs must be CUDA tensors")
    return _VariantFunction.apply(q.contiguous(), k.contiguous(), v.contiguous(),
                                  None if mask is None else mask.contiguous(),
                                  None if bias is None else bias.contiguous(), swap)


def _desc(q, B, L, H, D, mask, bias, swap, path="auto", dbias_dtype=None):
    if q.dtype not in _DT:
        raise N.ValidationError(f"unsupported dtype {q.dtype}")
    d = N.Desc(1, B, L, H, D, _DT[q.dtype], 1.0 / math.sqrt(D), int(mask is not None),
               int(bias is not None), _DT[dbias_dtype] if dbias_dtype is not None else N.EVO_F32,
               _PATHS[path])
    d.axes_swapped = int(swap)
    d.check_numerics = int(numeric_checks())
    return d


def _dims(q, swap):
    A0, A1, H, D = q.shape
    return (A1, A0, H, D) if swap else (A0, A1, H, D)


class _VariantFunction(torch.autograd.Function):
    """Raw-layout autograd: forward and backward both read/write the model's axes in place."""

    @staticmethod
    def forward(ctx, q, k, v, mask, bias, swap):
        B, L, H, D = _dims(q, swap)
        lib = N.load()
        d = _desc(q, B, L, H, D, mask, bias, swap)
        o = torch.empty_like(q)
        lse = torch.empty((B, H, L), device=q.device, dtype=torch.float32)
        wsb = lib.evo_attn_fwd_workspace_size(d)
        ws = torch.empty(max(wsb, 1), device=q.device, dtype=torch.uint8)
        N.check(lib.evo_attn_fwd(d, _ptr(q), _ptr(k), _ptr(v), _ptr(mask), _ptr(bias), _ptr(o),
                                 _ptr(lse), _ptr(ws), wsb, _stream()))
        ctx.save_for_backward(q, k, v, o, lse, mask, bias)
        ctx.swap = swap
        return o

    @staticmethod
    def backward(ctx, grad_o):
        q, k, v, o, lse, mask, bias = ctx.saved_tensors
        swap = ctx.swap
        B, L, H, D = _dims(q, swap)
        lib = N.load()
        d = _desc(q, B, L, H, D, mask, bias, swap, dbias_dtype=q.dtype)
        db1 = torch.empty_like(mask) if mask is not None and ctx.needs_input_grad[3] else None
        db2 = torch.empty_like(bias) if bias is not None and ctx.needs_input_grad[4] else None
        d.need_dbias1 = int(db1 is not None)
        dq, dk, dv = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
        wsb = lib.evo_attn_bwd_workspace_size(d)
        ws = torch.empty(max(wsb, 1), device=q.device, dtype=torch.uint8)
        N.check(lib.evo_attn_bwd(d, _ptr(grad_o.contiguous()), _ptr(q), _ptr(k), _ptr(v), _ptr(mask),
                                 _ptr(bias), _ptr(o), _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv),
                                 _ptr(db1), _ptr(db2), 0, _ptr(ws), wsb, _stream()))
        return dq, dk, dv, db1, db2, None


@torch.no_grad()
def variant_forward(variant, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                    bias: Optional[torch.Tensor] = None, mask: Optional[torch.Tensor] = None,
                    path: str = "auto") -> Tuple[torch.Tensor, torch.Tensor]:
    """Inference forward of one variant on raw (model-axis) contiguous Q/K/V with no layout copy.
    Returns (O in the raw axes, LSE [B, H, L] canonical fp32)."""
    variant = _as_variant(variant)
    swap = variant in (AttentionVariant.MsaColumnWise, AttentionVariant.TriangularEndNode)
    perm = _SWAP if swap else _IDENT
    qc, kc, vc = (t.permute(*perm) for t in (q, k, v))
    validate_variant_problem(variant, qc, kc, vc, bias, mask)
    for t in (q, k, v, bias, mask):
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise N.ValidationError("inputs must be contiguous CUDA tensors")
    B, L, H, D = qc.shape
    lib = N.load()
    d = _desc(q, B, L, H, D, mask, bias, swap, path)
    o = torch.empty_like(q)
    lse = torch.empty((B, H, L), device=q.device, dtype=torch.float32)
    wsb = lib.evo_attn_fwd_workspace_size(d)
    ws = torch.empty(max(wsb, 1), device=q.device, dtype=torch.uint8)
    N.check(lib.evo_attn_fwd(d, _ptr(q), _ptr(k), _ptr(v), _ptr(mask), _ptr(bias), _ptr(o),
                             _ptr(lse), _ptr(ws), wsb, _stream()))
    return o, lse


@torch.no_grad()
def chunked_forward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                    bias1: Optional[torch.Tensor] = None, bias2: Optional[torch.Tensor] = None,
                    chunk_rows: int = 64, scale: Optional[float] = None,
                    ) -> Tuple[torch.Tensor, torch.Tensor]:
    """Inference forward over row chunks of [Bo, N, L, H, D] inputs (OpenFold's chunked mode):
    each call covers `chunk_rows` MSA rows / start nodes of one outer batch, writing into one
    output buffer. Returns (O [Bo, N, L, H, D], LSE [Bo·N, H, L]) identical in layout to
    evoformer_attention_forward."""
    if chunk_rows < 1:
        raise N.ValidationError(f"chunk_rows must be >= 1, got {chunk_rows}")
    if q.dim() != 5:
        raise N.ValidationError(f"chunked_forward expects [Bo, N, L, H, D], got {tuple(q.shape)}")
    Bo, Nr, L, H, D = q.shape
    out = torch.empty_like(q)
    lse = torch.empty((Bo * Nr, H, L), dtype=torch.float32, device=q.device)
    for ob in range(Bo):
        b2 = None if bias2 is None else bias2[ob:ob + 1]
        for n0 in range(0, Nr, chunk_rows):
            n1 = min(Nr, n0 + chunk_rows)
            sl = lambda t: t[ob:ob + 1, n0:n1].contiguous()
            o, l = evoformer_attention_forward(sl(q), sl(k), sl(v),
                                               None if bias1 is None else sl(bias1), b2, scale)
            out[ob, n0:n1] = o[0]
            lse[ob * Nr + n0: ob * Nr + n1] = l
    return out, lse
