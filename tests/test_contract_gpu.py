"""GPU tests of the reference contract at the boundary:
  * NumericError (attention_tiled.cpp:49-65, 125-127, 209): NaN in Q / K / V / bias / dO and rows
    without a finite logit raise through the C-ABI, the operator API and DS4Sci_EvoformerAttention;
  * AccumPolicy::deterministic (attention_tiled.hpp:35-44, attention_tiled.cpp:246-252; SPEC.md:211
    "two runs are bit-identical"): the backward twice in deterministic mode is bitwise equal, on the
    tcgen05 path (single and chunked query axis, dBias1, raw layout, row windows) and the SIMT path;
  * DS4Sci_EvoformerAttention autograd: gradients of Q, K, V, bias1, bias2 against the oracle;
  * path resolution per direction, explicit tcgen05 requests outside the backward envelope, scales
    outside the 16-bit operand range, long-L forward without a bias1 staging budget.
"""
import math

import numpy as np
import pytest
import torch

from tests.util import TOL, make_inputs, nmax_err, oracle_fwd_bwd

pytestmark = pytest.mark.gpu

TD = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def _t(a, dtype="bf16"):
    return None if a is None else torch.tensor(a, dtype=TD[dtype], device="cuda")


# ------------------------------------------------------------------------------ NumericError
@pytest.mark.parametrize("where", ["q", "k", "v", "bias2"])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_nan_input_raises_numeric_error_forward(where, dtype):
    import paper_2310_04610_b200 as E

    q, k, v, do, b1, b2 = make_inputs(1, 3, 96, 2, 32, dtype=dtype, seed=1)
    arrs = {"q": q, "k": k, "v": v, "bias2": b2}
    arrs[where] = arrs[where].copy()
    arrs[where].reshape(-1)[arrs[where].size // 3] = np.nan
    with pytest.raises(E.NumericError):
        E.evoformer_attention_forward(_t(arrs["q"], dtype), _t(arrs["k"], dtype), _t(arrs["v"], dtype),
                                      _t(b1, dtype), _t(arrs["bias2"], dtype))


def test_nan_dout_raises_numeric_error_backward():
    import paper_2310_04610_b200 as E

    q, k, v, do, b1, b2 = make_inputs(1, 3, 128, 2, 32, seed=2)
    tq, tk, tv, tb1, tb2 = map(_t, (q, k, v, b1, b2))
    o, lse = E.evoformer_attention_forward(tq, tk, tv, tb1, tb2)
    bad = do.copy()
    bad[0, 1, 5, 1, 3] = np.nan
    with pytest.raises(E.NumericError):
        E.evoformer_attention_backward(_t(bad), tq, tk, tv, o, lse, tb1, tb2)
    # clean inputs after a failed call: the flag is per call
    E.evoformer_attention_backward(_t(do), tq, tk, tv, o, lse, tb1, tb2)


def test_row_without_finite_logit_raises():
    import paper_2310_04610_b200 as E

    q, k, v, do, b1, b2 = make_inputs(1, 2, 64, 2, 32, seed=3)
    b1 = b1.copy()
    b1[0, 1] = -np.inf  # every key of row 1 masked with -inf: the reference's non-finite logits
    with pytest.raises(E.NumericError):
        E.evoformer_attention_forward(_t(q), _t(k), _t(v), _t(b1), _t(b2))


def test_numeric_error_through_the_c_abi_and_ds4sci():
    import paper_2310_04610_b200 as E
    from paper_2310_04610_b200 import _native as N
    from paper_2310_04610_b200.evoformer_attention import make_desc

    q, k, v, do, b1, b2 = make_inputs(1, 2, 64, 2, 32, seed=4)
    q[0, 0, 0, 0, 0] = np.nan
    tq, tk, tv, tb1, tb2 = map(_t, (q, k, v, b1, b2))
    lib = N.load()
    d = make_desc(tq, tb1, tb2, None, check_numerics=True)
    ws = torch.empty(lib.evo_attn_fwd_workspace_size(d), dtype=torch.uint8, device="cuda")
    o, lse = torch.empty_like(tq), torch.empty(2, 2, 64, device="cuda")
    st = lib.evo_attn_fwd(d, tq.data_ptr(), tk.data_ptr(), tv.data_ptr(), tb1.data_ptr(), tb2.data_ptr(),
                          o.data_ptr(), lse.data_ptr(), ws.data_ptr(), ws.numel(),
                          torch.cuda.current_stream().cuda_stream)
    assert st == N.EVO_ERR_NUMERIC and "NaN" in lib.evo_attn_last_error().decode()
    d.check_numerics = 0  # unchecked calls are asynchronous and report nothing
    st = lib.evo_attn_fwd(d, tq.data_ptr(), tk.data_ptr(), tv.data_ptr(), tb1.data_ptr(), tb2.data_ptr(),
                          o.data_ptr(), lse.data_ptr(), ws.data_ptr(), ws.numel(),
                          torch.cuda.current_stream().cuda_stream)
    assert st == N.EVO_OK
    with pytest.raises(E.NumericError):
        E.DS4Sci_EvoformerAttention(tq, tk, tv, [tb1, tb2])
    prev = E.set_numeric_checks(False)
    try:
        E.DS4Sci_EvoformerAttention(tq, tk, tv, [tb1, tb2])  # no check, no raise
    finally:
        E.set_numeric_checks(prev)


# ------------------------------------------------------------------------------ determinism
def _bwd(inp, dtype, det, need_dbias1=False, path="auto", swapped=False):
    import paper_2310_04610_b200 as E

    q, k, v, do, b1, b2 = (_t(a, dtype) for a in inp)
    o, lse = E.evoformer_attention_forward(q, k, v, b1, b2, path=path)
    r = E.evoformer_attention_backward(do, q, k, v, o, lse, b1, b2, need_dbias1=need_dbias1,
                                       deterministic=det, path=path)
    torch.cuda.synchronize()
    return [x for x in r if x is not None]


@pytest.mark.parametrize("shape,dtype,need_dbias1,path", [
    ((1, 64, 384, 4, 32), "bf16", False, "auto"),   # tcgen05, one query chunk, 6 key tiles (C4-like)
    ((1, 24, 640, 2, 32), "bf16", False, "auto"),   # tcgen05, chunked query axis (dK/dV partials)
    ((2, 5, 256, 2, 16), "f16", True, "auto"),      # tcgen05 dBias1 partials, outer batch
    ((1, 200, 128, 1, 32), "bf16", False, "auto"),  # flat (non-aligned) CTA split: ordered strip flushes
    ((1, 8, 130, 2, 32), "bf16", True, "auto"),     # SIMT backward (L % 8 != 0)
    ((1, 32, 64, 8, 32), "f32", True, "auto"),      # SIMT fp32 (config 1)
])
def test_deterministic_backward_is_bitwise_reproducible(shape, dtype, need_dbias1, path):
    inp = make_inputs(*shape, dtype=dtype, seed=21)
    a = _bwd(inp, dtype, True, need_dbias1, path)
    b = _bwd(inp, dtype, True, need_dbias1, path)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    # and it is the same operator: parity with the oracle and with the default (unordered) mode
    want = oracle_fwd_bwd(*inp, need_dbias1=need_dbias1)
    names = ["dQ", "dK", "dV"] + (["dBias1"] if need_dbias1 else []) + ["dBias2"]
    wants = list(want[2:5]) + ([want[5]] if need_dbias1 else []) + [want[6]]
    fast = _bwd(inp, dtype, False, need_dbias1, path)
    for n, g, w, f in zip(names, a, wants, fast):
        assert nmax_err(g.float().cpu().numpy(), w) <= TOL[dtype], n
        assert nmax_err(g.float().cpu().numpy(), f.float().cpu().numpy()) <= 1e-2, n


def test_deterministic_row_windows(monkeypatch):
    # several deterministic row windows per outer batch (partials bounded per window; the last one
    # ragged) run in order: the result stays bitwise reproducible and equal to the unordered mode
    monkeypatch.setenv("EVO_DET_WINDOW_ROWS", "2")  # the C-ABI sizes windows of at most 2 rows
    inp = make_inputs(2, 5, 640, 1, 32, dtype="bf16", seed=5)
    a = _bwd(inp, "bf16", True)
    b = _bwd(inp, "bf16", True)
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    fast = _bwd(inp, "bf16", False)
    for x, f in zip(a, fast):
        assert nmax_err(x.float().cpu().numpy(), f.float().cpu().numpy()) <= 1e-2


def test_deterministic_raw_layout_variant():
    import paper_2310_04610_b200 as E
    from paper_2310_04610_b200 import _native as N
    from paper_2310_04610_b200.variants import _desc

    g = torch.Generator(device="cuda").manual_seed(3)
    L, Nr, H, D = 256, 48, 2, 32
    r = lambda *s: (torch.rand(*s, generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    q, k, v, do = (r(L, Nr, H, D) for _ in range(4))
    bias = r(H, L, L)
    lib = N.load()

    def run():
        d = _desc(q, Nr, L, H, D, None, bias, True)
        o, lse = torch.empty_like(q), torch.empty(Nr, H, L, device="cuda")
        ws = torch.empty(lib.evo_attn_fwd_workspace_size(d), dtype=torch.uint8, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        N.check(lib.evo_attn_fwd(d, q.data_ptr(), k.data_ptr(), v.data_ptr(), None, bias.data_ptr(),
                                 o.data_ptr(), lse.data_ptr(), ws.data_ptr(), ws.numel(), s))
        d.deterministic = 1
        wsb = lib.evo_attn_bwd_workspace_size(d)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        out = [torch.empty_like(q) for _ in range(3)] + [torch.empty(H, L, L, device="cuda")]
        N.check(lib.evo_attn_bwd(d, do.data_ptr(), q.data_ptr(), k.data_ptr(), v.data_ptr(), None, bias.data_ptr(),
                                 o.data_ptr(), lse.data_ptr(), *(t.data_ptr() for t in out[:3]), None,
                                 out[3].data_ptr(), 0, ws.data_ptr(), wsb, s))
        torch.cuda.synchronize()
        return out

    a, b = run(), run()
    for x, y in zip(a, b):
        assert torch.equal(x, y)


# ------------------------------------------------------------------------------ DS4Sci autograd
@pytest.mark.parametrize("shape", [(1, 6, 96, 2, 32), (2, 3, 200, 2, 16)])
def test_ds4sci_autograd_all_gradients(shape):
    import paper_2310_04610_b200 as E

    q, k, v, do, b1, b2 = make_inputs(*shape, dtype="bf16", seed=8)
    tq, tk, tv, tb1, tb2 = (_t(a).requires_grad_(True) for a in (q, k, v, b1, b2))
    o = E.DS4Sci_EvoformerAttention(tq, tk, tv, [tb1, tb2])
    o.backward(_t(do))
    want = oracle_fwd_bwd(q, k, v, do, b1, b2, need_dbias1=True)
    got = [o.detach(), tq.grad, tk.grad, tv.grad, tb1.grad, tb2.grad]
    wants = [want[0], want[2], want[3], want[4], want[5], want[6]]
    for name, g, w in zip(["O", "dQ", "dK", "dV", "dBias1", "dBias2"], got, wants):
        assert g is not None and g.shape == tuple(w.shape), name
        # gradients come back in the input dtype (bf16), one more rounding than the fp32 outputs
        assert nmax_err(g.float().cpu().numpy(), w) <= 1.5e-2, name


def test_ds4sci_biases_optional():
    import paper_2310_04610_b200 as E

    q, k, v, do, b1, b2 = make_inputs(1, 3, 64, 2, 32, dtype="bf16", seed=9, bias2=False)
    tq, tk, tv = (_t(a).requires_grad_(True) for a in (q, k, v))
    tb1 = _t(b1)
    o = E.DS4Sci_EvoformerAttention(tq, tk, tv, [tb1])  # mask only (MSA column attention)
    o.backward(_t(do))
    want = oracle_fwd_bwd(q, k, v, do, b1, None)
    assert nmax_err(o.detach().float().cpu().numpy(), want[0]) <= 1e-2
    assert nmax_err(tq.grad.float().cpu().numpy(), want[2]) <= 1.5e-2
    with pytest.raises(E.ValidationError):
        E.DS4Sci_EvoformerAttention(tq, tk, tv, [tb1, None, None])


# ------------------------------------------------------------------------------ envelopes
def test_resolved_path_per_direction_and_explicit_tcgen05():
    import paper_2310_04610_b200 as E

    q = torch.zeros(1, 2, 64, 2, 64, dtype=torch.bfloat16, device="cuda")
    assert E.resolved_path(q) == "tcgen05"
    assert E.resolved_path(q, direction="bwd") == "simt"  # D = 64 backward runs on the SIMT kernels
    assert E.resolved_path(q, path="tcgen05", direction="bwd") == "invalid"
    o, lse = E.evoformer_attention_forward(q, q, q, path="tcgen05")
    with pytest.raises(E.UnsupportedError):
        E.evoformer_attention_backward(q, q, q, q, o, lse, path="tcgen05")


def test_scale_outside_16bit_operands_takes_simt():
    import paper_2310_04610_b200 as E

    q, k, v, do, b1, b2 = make_inputs(1, 2, 64, 2, 32, dtype="f16", seed=6)
    tq = _t(q, "f16")
    from paper_2310_04610_b200 import _native as N
    from paper_2310_04610_b200.evoformer_attention import make_desc

    lib = N.load()
    assert lib.evo_attn_resolved_path(make_desc(tq, None, None, 1e-6)) == N.EVO_PATH_SIMT  # 1/scale > f16 max
    assert lib.evo_attn_resolved_path(make_desc(tq, None, None, 0.0)) == N.EVO_PATH_SIMT
    o, lse = E.evoformer_attention_forward(tq, _t(k, "f16"), _t(v, "f16"), scale=1e-6)
    assert torch.isfinite(o.float()).all()


def test_long_l_forward_without_bias1_staging():
    # L = 6016: the forward no longer reserves shared memory for bias1 rows it does not stage (the
    # UMMA warp reads them from global), so long triangle / column attention stays on tcgen05
    import paper_2310_04610_b200 as E
    from tests.util import O

    L, H, D = 6016, 1, 32
    q, k, v, _, b1, b2 = make_inputs(1, 1, L, H, D, dtype="bf16", seed=12)
    tq, tk, tv, tb1, tb2 = map(_t, (q, k, v, b1, b2))
    assert E.resolved_path(tq, tb1, tb2) == "tcgen05"
    o, lse = E.evoformer_attention_forward(tq, tk, tv, tb1, tb2)
    torch.cuda.synchronize()
    p = O.Problem(1, L, H, D, fmt=O.F32)
    r = lambda a: a.reshape(-1).astype(np.float64)
    wo, wl = O.forward(p, r(q), r(k), r(v), r(b1), r(b2))
    assert nmax_err(o.float().cpu().numpy(), wo.reshape(q.shape)) <= 1e-2
    assert nmax_err(lse.cpu().numpy(), wl.transpose(1, 0, 2)) <= 1e-2


# ------------------------------------------------------------------------------ bounded workspace
@pytest.mark.parametrize("shape", [(1, 7, 640, 2, 32), (2, 5, 256, 2, 32)])
def test_windowed_accumulators(monkeypatch, shape):
    # the default (unordered) backward bounds its fp32 accumulators to one row window at a time when the
    # whole problem's would exceed the cap (C5); forced here to windows of 2 rows (ragged last window,
    # chunked and unchunked query axis, outer batch) — same results as the oracle
    import paper_2310_04610_b200 as E

    inp = make_inputs(*shape, dtype="bf16", seed=31)
    monkeypatch.setenv("EVO_BWD_WINDOW_ROWS", "2")
    got = _bwd(inp, "bf16", False)
    want = oracle_fwd_bwd(*inp)
    for name, g, w in zip(["dQ", "dK", "dV", "dBias2"], got, [want[2], want[3], want[4], want[6]]):
        assert nmax_err(g.float().cpu().numpy(), w) <= TOL["bf16"], name
    monkeypatch.delenv("EVO_BWD_WINDOW_ROWS")
    q = _t(inp[0])
    from paper_2310_04610_b200 import _native as N
    from paper_2310_04610_b200.evoformer_attention import make_desc

    lib = N.load()
    d = make_desc(q, _t(inp[4]), _t(inp[5]), None)
    full = lib.evo_attn_bwd_workspace_size(d)
    monkeypatch.setenv("EVO_BWD_WINDOW_ROWS", "2")
    assert lib.evo_attn_bwd_workspace_size(d) < full
