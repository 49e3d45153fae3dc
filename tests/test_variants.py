"""Variant layer (msa_row / msa_col / tri_start / tri_end) and the chunked inference forward.

Host logic (names, validation, canonical layouts; attention.cpp:10-32, 48-124, 160-166) runs on
CPU; the `gpu` tests check each variant end to end against the oracle on the canonical problem,
with the north-star tolerance (bf16 1e-2 normalised max error).
"""
import numpy as np
import pytest
import torch

import paper_2310_04610_b200 as E
from paper_2310_04610_b200 import variants as Vr
from tests.util import TOL, make_inputs, nmax_err, oracle_fwd_bwd


def test_variant_names_round_trip():
    for v in Vr.AttentionVariant:
        assert Vr.variant_from_name(Vr.variant_name(v)) is v
    assert not Vr.variant_has_bias(Vr.AttentionVariant.MsaColumnWise)
    assert all(Vr.variant_has_bias(v) for v in Vr.AttentionVariant if v.value != "msa_col")
    with pytest.raises(E.ValidationError, match="unknown attention variant"):
        Vr.variant_from_name("msa_diag")


def test_layout_from_msa_permutations():
    raw = torch.arange(3 * 5 * 2 * 4, dtype=torch.float32).reshape(3, 5, 2, 4)
    row = Vr.layout_from_msa("msa_row", raw)
    assert row.permutation == (0, 1, 2, 3) and (row.batch_extent, row.attended_extent) == (3, 5)
    assert torch.equal(row.tensor, raw)
    col = Vr.layout_from_msa("msa_col", raw)
    assert col.permutation == (1, 0, 2, 3) and (col.batch_extent, col.attended_extent) == (5, 3)
    assert col.tensor.is_contiguous() and torch.equal(col.tensor[2, 1], raw[1, 2])
    assert torch.equal(col.tensor.permute(*Vr.inverse_permutation(col.permutation)), raw)
    with pytest.raises(E.ValidationError, match="rank-4"):
        Vr.layout_from_msa("tri_end", raw[0])


def test_variant_validation_taxonomy():
    q = torch.zeros(4, 6, 2, 8)
    bias = torch.zeros(2, 6, 6)
    with pytest.raises(E.ValidationError, match="requires a bias"):
        Vr.validate_variant_problem("msa_row", q, q, q)
    with pytest.raises(E.ValidationError, match="does not take a bias"):
        Vr.validate_variant_problem("msa_col", q, q, q, bias)
    with pytest.raises(E.ValidationError, match="B == L"):
        Vr.validate_variant_problem("tri_start", q, q, q, bias)
    with pytest.raises(E.ValidationError, match=r"bias must be \(H, L, L\)"):
        Vr.validate_variant_problem("msa_row", q, q, q, torch.zeros(2, 6, 5))
    with pytest.raises(E.ValidationError, match="mask must be"):
        Vr.validate_variant_problem("msa_row", q, q, q, bias, torch.zeros(6, 4))
    with pytest.raises(E.ValidationError, match="share one shape"):
        Vr.validate_variant_problem("msa_col", q, q[:, :5], q)
    with pytest.raises(E.NumericError, match="finite"):
        Vr.validate_variant_problem("msa_row", q, q, q, bias, scale=float("inf"))
    Vr.validate_variant_problem("tri_end", torch.zeros(6, 6, 2, 8), torch.zeros(6, 6, 2, 8),
                                torch.zeros(6, 6, 2, 8), bias)
    with pytest.raises(E.ValidationError, match="chunk_rows"):
        Vr.chunked_forward(torch.zeros(1, 2, 8, 1, 8), None, None, chunk_rows=0)


# ---------------------------------------------------------------- GPU parity of the variants

def _variant_case(variant, raw_shape, dtype="bf16", seed=3):
    """Raw (model-axis) inputs for `variant` and the oracle on the canonical problem."""
    A0, A1, H, D = raw_shape
    swap = variant in ("msa_col", "tri_end")
    B, L = (A1, A0) if swap else (A0, A1)
    q, k, v, do, b1, b2 = make_inputs(1, B, L, H, D, dtype=dtype, bias1=True,
                                      bias2=Vr.variant_has_bias(Vr.variant_from_name(variant)), seed=seed)
    want = oracle_fwd_bwd(q, k, v, do, b1, b2)
    to_raw = (lambda a: a[0].transpose(1, 0, 2, 3)) if swap else (lambda a: a[0])
    raw = [to_raw(a) for a in (q, k, v, do)]
    return raw, b1, b2, want, to_raw


@pytest.mark.gpu
@pytest.mark.parametrize("variant,raw_shape", [
    ("msa_row", (16, 128, 4, 32)),
    ("msa_col", (64, 96, 4, 32)),       # attends over N_msa = 64 for each of 96 residues
    ("tri_start", (96, 96, 2, 32)),
    ("tri_end", (96, 96, 2, 32)),
    ("tri_end", (100, 100, 2, 32)),     # L % 8 != 0: SIMT backward in the raw layout
    ("msa_col", (200, 24, 2, 16)),      # ragged tiles, D 16
])
def test_variant_parity(variant, raw_shape, cuda):
    raw, b1, b2, want, to_raw = _variant_case(variant, raw_shape)
    dev = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.bfloat16, device="cuda")
    q, k, v, do = (dev(a).requires_grad_(i < 3) for i, a in enumerate(raw))
    B, L = b1.shape[1], b1.shape[4]
    mask = dev(b1.reshape(B, L)).requires_grad_(False)
    bias = None if b2 is None else dev(b2.reshape(b2.shape[2:])).requires_grad_(True)
    o = Vr.variant_attention(variant, q, k, v, bias, mask)
    o.backward(do)
    torch.cuda.synchronize()
    wo, _, wdq, wdk, wdv, _, wdb2 = want
    f = lambda t: t.detach().float().cpu().numpy()
    errs = {"O": nmax_err(f(o), to_raw(wo)), "dQ": nmax_err(f(q.grad), to_raw(wdq)),
            "dK": nmax_err(f(k.grad), to_raw(wdk)), "dV": nmax_err(f(v.grad), to_raw(wdv))}
    if bias is not None:
        errs["dBias2"] = nmax_err(f(bias.grad), wdb2.reshape(bias.shape))
    assert max(errs.values()) <= TOL["bf16"], errs


@pytest.mark.gpu
@pytest.mark.parametrize("chunk_rows", [1, 5, 64])
def test_chunked_forward_matches_full(chunk_rows, cuda):
    q, k, v, _, b1, b2 = make_inputs(2, 12, 128, 4, 32, dtype="bf16", seed=5)
    dev = lambda a: torch.tensor(a, dtype=torch.bfloat16, device="cuda")
    tq, tk, tv, tb1, tb2 = map(dev, (q, k, v, b1, b2))
    o_full, lse_full = E.evoformer_attention_forward(tq, tk, tv, tb1, tb2)
    o, lse = Vr.chunked_forward(tq, tk, tv, tb1, tb2, chunk_rows=chunk_rows)
    torch.cuda.synchronize()
    # rows are independent: a chunk's kernels compute the same row the same way
    assert (o.float() - o_full.float()).abs().max().item() <= 1e-2 * o_full.float().abs().max().item()
    assert (lse - lse_full).abs().max().item() <= 1e-4 * lse_full.abs().max().item()
    wo, wlse = oracle_fwd_bwd(q, k, v, q, b1, b2)[:2]
    assert nmax_err(o.float().cpu().numpy(), wo) <= TOL["bf16"]


@pytest.mark.gpu
@pytest.mark.parametrize("variant,raw_shape,path", [
    ("msa_col", (64, 96, 4, 32), "tcgen05"),
    ("tri_end", (96, 96, 2, 32), "tcgen05"),
    ("tri_end", (136, 136, 2, 32), "tcgen05"),  # ragged query and key tiles (L = 136)
    ("tri_end", (96, 96, 2, 32), "simt"),
    ("tri_start", (96, 96, 2, 32), "auto"),
])
def test_variant_forward_in_place_layout(variant, raw_shape, path, cuda):
    """Copy-free forward: the kernels read the raw msa_col / tri_end layout through the swapped
    strides and write O back in it; parity against the oracle on the canonical problem."""
    raw, b1, b2, want, to_raw = _variant_case(variant, raw_shape)
    dev = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.bfloat16, device="cuda")
    q, k, v = (dev(a) for a in raw[:3])
    B, L = b1.shape[1], b1.shape[4]
    mask = dev(b1.reshape(B, L))
    bias = None if b2 is None else dev(b2.reshape(b2.shape[2:]))
    o, lse = Vr.variant_forward(variant, q, k, v, bias, mask, path=path)
    torch.cuda.synchronize()
    assert o.shape == q.shape
    wo, wlse = want[0], want[1]
    assert nmax_err(o.float().cpu().numpy(), to_raw(wo)) <= TOL["bf16"]
    assert nmax_err(lse.cpu().numpy(), wlse.reshape(lse.shape)) <= TOL["bf16"]
    # same numbers as the transposing autograd path
    o2 = Vr.variant_attention(variant, q, k, v, bias, mask)
    assert (o.float() - o2.float()).abs().max().item() <= 2e-2 * o2.float().abs().max().item()


@pytest.mark.gpu
def test_variant_msa_col_mask_grad_chunked(cuda):
    """msa_col in the raw layout with a mask gradient: the tcgen05 backward splits the query axis
    (L = 320, three tiles -> chunks of two), reduces dK/dV in canonical fp32 accumulators and the
    conversion writes them back in the raw layout."""
    A0, A1, H, D = 320, 16, 2, 32
    q, k, v, do, b1, _ = make_inputs(1, A1, A0, H, D, dtype="bf16", bias1=True, bias2=False, seed=9)
    want = oracle_fwd_bwd(q, k, v, do, b1, None, need_dbias1=True)
    to_raw = lambda a: a[0].transpose(1, 0, 2, 3)
    dev = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.bfloat16, device="cuda")
    tq, tk, tv, tdo = (dev(to_raw(a)).requires_grad_(i < 3) for i, a in enumerate((q, k, v, do)))
    mask = dev(b1.reshape(A1, A0)).requires_grad_(True)
    o = Vr.variant_attention("msa_col", tq, tk, tv, None, mask)
    o.backward(tdo)
    torch.cuda.synchronize()
    f = lambda t: t.detach().float().cpu().numpy()
    wo, _, wdq, wdk, wdv, wdb1, _ = want
    errs = {"O": nmax_err(f(o), to_raw(wo)), "dQ": nmax_err(f(tq.grad), to_raw(wdq)),
            "dK": nmax_err(f(tk.grad), to_raw(wdk)), "dV": nmax_err(f(tv.grad), to_raw(wdv)),
            "dBias1": nmax_err(f(mask.grad), wdb1.reshape(A1, A0))}
    assert max(errs.values()) <= TOL["bf16"], errs
