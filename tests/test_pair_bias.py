"""Pair-bias projection: LayerNorm(z)·W → bias2 in the attention's [Bo, 1, H, L, L]
layout, and its backward from dBias2 in that layout. Reference: the fp32 torch composition
(layer_norm → linear → permute) on the same 16-bit-rounded z — a floating-point kernel, so a torch
fp32 reference (the reference repo has no counterpart)."""
import pytest
import torch

import paper_2310_04610_b200 as E
from paper_2310_04610_b200 import _native as N

gpu = pytest.mark.gpu


def _ref(z, g, b, w, eps):
    y = torch.nn.functional.layer_norm(z.float(), (z.shape[-1],), g.float(), b.float(), eps)
    return (y @ w.float().t()).permute(0, 3, 1, 2).unsqueeze(1)  # [Bo, 1, H, L, L]


def _inputs(Bo, L, cz, H, dtype, seed=0):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    r = lambda *s: torch.randn(*s, generator=gen, device="cuda")
    z = (r(Bo, L, L, cz) * 2 + 0.5).to(dtype)
    g = 1 + 0.1 * r(cz)
    b = 0.1 * r(cz)
    w = r(H, cz) / cz ** 0.5
    return z, g, b, w


def _nerr(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-30)).item()


@gpu
@pytest.mark.parametrize("Bo,L,cz,H,dtype", [(1, 64, 128, 8, torch.bfloat16), (2, 45, 64, 4, torch.float16),
                                            (1, 130, 256, 16, torch.bfloat16), (1, 33, 32, 3, torch.bfloat16)])
def test_forward_matches_torch(Bo, L, cz, H, dtype):
    z, g, b, w = _inputs(Bo, L, cz, H, dtype)
    out = E.pair_bias_forward(z, g, b, w)
    assert out.shape == (Bo, 1, H, L, L) and out.dtype == dtype
    assert _nerr(out, _ref(z, g, b, w, 1e-5)) < 1e-2


@gpu
@pytest.mark.parametrize("Bo,L,cz,H,dtype,gdtype", [(1, 64, 128, 8, torch.bfloat16, torch.float32),
                                                   (2, 45, 64, 4, torch.float16, torch.float16),
                                                   (1, 70, 256, 12, torch.bfloat16, torch.bfloat16)])
def test_backward_matches_torch_autograd(Bo, L, cz, H, dtype, gdtype):
    z, g, b, w = _inputs(Bo, L, cz, H, dtype, seed=1)
    gen = torch.Generator(device="cuda").manual_seed(5)
    dbias = torch.randn(Bo, 1, H, L, L, generator=gen, device="cuda").to(gdtype)
    zr = z.float().requires_grad_()
    gr, br, wr = (t.clone().requires_grad_() for t in (g, b, w))
    _ref(zr, gr, br, wr, 1e-5).backward(dbias.float())
    dz, dg, db, dw = E.pair_bias_backward(dbias, z, g, b, w)
    assert dz.dtype == dtype and dw.shape == w.shape
    assert _nerr(dz, zr.grad) < 1e-2
    for got, want in ((dg, gr.grad), (db, br.grad), (dw, wr.grad)):
        assert _nerr(got, want) < 1e-4


@gpu
def test_autograd_chain_into_attention():
    """z → pair_bias → DS4Sci_EvoformerAttention → loss: gradients reach z and the projection's
    parameters through the attention's dBias2 (compared with the same chain in fp32 torch)."""
    Bo, Nr, L, H, D, cz = 1, 3, 48, 4, 32, 64
    gen = torch.Generator(device="cuda").manual_seed(3)
    r = lambda *s: torch.randn(*s, generator=gen, device="cuda")
    z, g, b, w = _inputs(Bo, L, cz, H, torch.bfloat16, seed=4)
    q, k, v = ((r(Bo, Nr, L, H, D) * 0.5).to(torch.bfloat16) for _ in range(3))
    wq = w.clone().requires_grad_()
    bias2 = E.pair_bias(z, g, b, wq)
    o = E.DS4Sci_EvoformerAttention(q, k, v, [None, bias2])
    o.float().square().sum().backward()
    # fp32 reference chain
    wr = w.clone().requires_grad_()
    b2 = _ref(z, g, b, wr, 1e-5)
    s = torch.einsum("bnihd,bnjhd->bnhij", q.float(), k.float()) / D ** 0.5 + b2
    orf = torch.einsum("bnhij,bnjhd->bnihd", s.softmax(-1), v.float())
    orf.square().sum().backward()
    assert _nerr(wq.grad, wr.grad) < 2e-2


@gpu
def test_validation():
    z = torch.zeros(1, 8, 8, 48, device="cuda", dtype=torch.bfloat16)  # c_z not a multiple of 32
    with pytest.raises(N.UnsupportedError):
        E.pair_bias_forward(z, torch.ones(48, device="cuda"), torch.zeros(48, device="cuda"),
                            torch.zeros(4, 48, device="cuda"))
    with pytest.raises(N.ValidationError):
        E.pair_bias_forward(torch.zeros(1, 8, 8, 32, device="cuda"), torch.ones(32, device="cuda"),
                            torch.zeros(32, device="cuda"), torch.zeros(4, 32, device="cuda"))
