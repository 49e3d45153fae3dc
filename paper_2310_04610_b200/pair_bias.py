"""Pair-bias projection feeding the attention's bias2.

OpenFold's MSARowAttentionWithPairBias computes the pair bias as linear_z(layer_norm_z(z)) and
permutes it to [*, 1, H, N_res, N_res] before DS4Sci_EvoformerAttention. `pair_bias` does both in
one pass over z (csrc/pair_bias.cu) and writes the [Bo, 1, H, L, L] layout the attention kernels
read; its backward consumes the attention's dBias2 in that same layout (fp32 or 16-bit) — no
permute / contiguous copies and no rounding of dBias2 in between. The reference has no counterpart
(SPEC.md:153 lists projections as non-goals); parity is against the fp32 torch composition.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from .evoformer_attention import _DT


def _desc(z: torch.Tensor, H: int, eps: float, dbias_dtype: torch.dtype = torch.float32) -> N.PairBiasDesc:
    if z.dim() != 4 or z.shape[1] != z.shape[2]:
        raise N.ValidationError(f"z must be [Bo, L, L, c_z], got {tuple(z.shape)}")
    if z.dtype not in (torch.bfloat16, torch.float16):
        raise N.ValidationError("z must be bf16 or f16")
    d = N.PairBiasDesc()
    d.Bo, d.L, d.C, d.H = z.shape[0], z.shape[1], z.shape[3], H
    d.dtype = _DT[z.dtype]
    d.dbias_dtype = _DT[dbias_dtype]
    d.eps = float(eps)
    return d


def _f32(t: torch.Tensor) -> torch.Tensor:
    return t.detach().to(torch.float32).contiguous()


def pair_bias_forward(z: torch.Tensor, ln_weight: torch.Tensor, ln_bias: torch.Tensor, weight: torch.Tensor,
                      eps: float = 1e-5) -> torch.Tensor:
    """bias2 [Bo, 1, H, L, L] (z's dtype) = (LayerNorm(z; ln_weight, ln_bias, eps) @ weight.T) permuted.

    z [Bo, L, L, c_z] bf16/f16; weight [H, c_z] (nn.Linear(c_z, H, bias=False).weight); ln_* [c_z]."""
    lib = N.load()
    z = z.contiguous()
    H = weight.shape[0]
    d = _desc(z, H, eps)
    out = torch.empty((z.shape[0], 1, H, z.shape[1], z.shape[1]), device=z.device, dtype=z.dtype)
    w = _f32(weight).t().contiguous()  # [c_z, H]
    g, b = _f32(ln_weight), _f32(ln_bias)
    st = torch.cuda.current_stream(z.device).cuda_stream
    N.check(lib.evo_pair_bias_fwd(C.byref(d), z.data_ptr(), g.data_ptr(), b.data_ptr(), w.data_ptr(),
                                  out.data_ptr(), st))
    return out


def pair_bias_backward(dbias2: torch.Tensor, z: torch.Tensor, ln_weight: torch.Tensor, ln_bias: torch.Tensor,
                       weight: torch.Tensor, eps: float = 1e-5):
    """(dz, d_ln_weight, d_ln_bias, d_weight) from dBias2 [Bo, 1, H, L, L] (fp32, or z's dtype) — the
    attention backward's output layout. Weight gradients are fp32 sums in a fixed order."""
    lib = N.load()
    z = z.contiguous()
    H = weight.shape[0]
    if dbias2.dtype not in (torch.float32, z.dtype):
        dbias2 = dbias2.to(torch.float32)
    dbias2 = dbias2.contiguous()
    d = _desc(z, H, eps, dbias2.dtype)
    w = _f32(weight).t().contiguous()
    g, b = _f32(ln_weight), _f32(ln_bias)
    dz = torch.empty_like(z)
    cz = z.shape[3]
    dg = torch.empty(cz, device=z.device, dtype=torch.float32)
    db = torch.empty(cz, device=z.device, dtype=torch.float32)
    dw = torch.empty((cz, H), device=z.device, dtype=torch.float32)
    nws = lib.evo_pair_bias_bwd_workspace_size(C.byref(d))
    ws = torch.empty(max(nws, 1), device=z.device, dtype=torch.uint8)
    st = torch.cuda.current_stream(z.device).cuda_stream
    N.check(lib.evo_pair_bias_bwd(C.byref(d), dbias2.data_ptr(), z.data_ptr(), g.data_ptr(), b.data_ptr(),
                                  w.data_ptr(), dz.data_ptr(), dg.data_ptr(), db.data_ptr(), dw.data_ptr(),
                                  ws.data_ptr(), nws, st))
    return dz, dg, db, dw.t()


class PairBiasFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, z, ln_weight, ln_bias, weight, eps=1e-5):
        ctx.save_for_backward(z, ln_weight, ln_bias, weight)
        ctx.eps = eps
        return pair_bias_forward(z, ln_weight, ln_bias, weight, eps)

    @staticmethod
    def backward(ctx, dbias2):
        z, ln_weight, ln_bias, weight = ctx.saved_tensors
        dz, dg, db, dw = pair_bias_backward(dbias2, z, ln_weight, ln_bias, weight, ctx.eps)
        return dz, dg.to(ln_weight.dtype), db.to(ln_bias.dtype), dw.to(weight.dtype), None


def pair_bias(z, ln_weight, ln_bias, weight, eps: float = 1e-5) -> torch.Tensor:
    """Autograd form of pair_bias_forward: bias2 for DS4Sci_EvoformerAttention from the pair
    representation z (OpenFold layer_norm_z + linear_z + permute, fused)."""
    return PairBiasFunction.apply(z, ln_weight, ln_bias, weight, eps)
