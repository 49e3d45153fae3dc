"""GPU parity: the CUDA path (through the C-ABI) vs the oracle on identical inputs.

Bar (north star): fp32 within 1e-4, bf16/f16 within 1e-2 of the F32 oracle on
identically rounded inputs, normalized max-abs error, for O and all four
gradients (dQ, dK, dV, dBias2), plus LSE and dBias1.
"""
import numpy as np
import pytest
import torch

from tests.util import TOL, make_inputs, nmax_err, oracle_fwd_bwd, ref_rel_err

pytestmark = pytest.mark.gpu

TD = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def run_gpu(q, k, v, do, b1, b2, dtype, path="auto", need_dbias1=False, dbias_dtype=torch.float32):
    import paper_2310_04610_b200 as E

    t = lambda a: None if a is None else torch.tensor(a, dtype=TD[dtype], device="cuda")
    tq, tk, tv, tdo, tb1, tb2 = map(t, (q, k, v, do, b1, b2))
    o, lse = E.evoformer_attention_forward(tq, tk, tv, tb1, tb2, path=path)
    dq, dk, dv, db1, db2 = E.evoformer_attention_backward(
        tdo, tq, tk, tv, o, lse, tb1, tb2, need_dbias1=need_dbias1, dbias_dtype=dbias_dtype, path=path)
    torch.cuda.synchronize()
    n = lambda a: None if a is None else a.float().cpu().numpy()
    return tuple(map(n, (o, lse, dq, dk, dv, db1, db2)))


def check(shape, dtype, bias1=True, bias2=True, path="auto", need_dbias1=False, seed=0,
          dbias_dtype=torch.float32, tol=None):
    q, k, v, do, b1, b2 = make_inputs(*shape, dtype=dtype, bias1=bias1, bias2=bias2, seed=seed)
    got = run_gpu(q, k, v, do, b1, b2, dtype, path, need_dbias1, dbias_dtype)
    want = oracle_fwd_bwd(q, k, v, do, b1, b2, need_dbias1=need_dbias1)
    tol = tol or TOL[dtype]
    names = ["O", "LSE", "dQ", "dK", "dV", "dBias1", "dBias2"]
    report = {}
    for name, g, w in zip(names, got, want):
        if w is None:
            assert g is None or name == "dBias1", name
            continue
        assert g is not None, f"{name} missing"
        assert np.isfinite(g).all(), f"{name} has non-finite values"
        report[name] = (nmax_err(g, w), ref_rel_err(g, w))
    bad = {k_: v_ for k_, v_ in report.items() if v_[0] > tol}
    assert not bad, f"parity failed (tol {tol}): {bad}; all: {report}"
    return report


def test_config1_fp32_msa_row_mask_pair():
    # BASELINE configs[0]: B=1 N_seq=32 N_res=64 H=8 D=32 fp32, mask + pair bias
    check((1, 32, 64, 8, 32), "f32")


def test_bf16_edge_tiles_l130():
    # 130 exercises clipped edge tiles (attention_tiled.cpp:89,109; run.cpp:147)
    check((1, 4, 130, 2, 32), "bf16")


def test_bf16_no_bias_msa_col():
    check((1, 6, 96, 2, 32), "bf16", bias1=False, bias2=False)


def test_bf16_pair_bias_only_triangle():
    check((1, 48, 48, 4, 32), "bf16", bias1=False)


def test_bf16_outer_batch():
    check((2, 3, 72, 2, 32), "bf16")


def test_f16():
    check((1, 4, 100, 2, 32), "f16")


@pytest.mark.parametrize("D", [4, 8, 16, 64])
def test_head_dims(D):
    check((1, 3, 70, 2, D), "bf16")


@pytest.mark.parametrize("shape", [(1, 4, 128, 2, 8), (1, 8, 384, 4, 8), (2, 3, 200, 2, 8), (1, 2, 640, 2, 8)])
def test_d8_on_tcgen05(shape):
    # D = 8 (the reference's attn-bench shape family, run.cpp:137-157) runs the D = 16 tcgen05 kernels on
    # zero-padded TMA boxes: forward and backward (incl. chunked query axis, outer batch)
    import paper_2310_04610_b200 as E

    check(shape, "bf16", need_dbias1=shape[2] <= 384)
    q = torch.zeros(shape, dtype=torch.bfloat16, device="cuda")
    assert E.resolved_path(q) == "tcgen05"
    assert E.resolved_path(q, direction="bwd") == "tcgen05"


def test_fp32_small_d_reference_bench_shape():
    # the reference's attn-bench default (4,130,2,8) F32 (run.cpp:137-157)
    check((1, 4, 130, 2, 8), "f32")


def test_dbias1_and_bf16_dbias_output():
    check((1, 5, 64, 2, 32), "bf16", need_dbias1=True)
    check((1, 5, 64, 2, 32), "bf16", need_dbias1=True, dbias_dtype=torch.bfloat16, tol=1.5e-2)


def test_single_key_identity():
    # L=1 => O = V
    import paper_2310_04610_b200 as E

    q, k, v, *_ = make_inputs(1, 4, 1, 2, 32, dtype="bf16", bias1=False, bias2=False)
    tv = torch.tensor(v, dtype=torch.bfloat16, device="cuda")
    o, _ = E.evoformer_attention_forward(torch.tensor(q, dtype=torch.bfloat16, device="cuda"),
                                         torch.tensor(k, dtype=torch.bfloat16, device="cuda"), tv)
    assert torch.equal(o, tv)


@pytest.mark.parametrize("path", ["simt", "auto"])
def test_paths_agree(path):
    check((1, 2, 128, 2, 32), "bf16", path=path)


def test_launches_counted():
    import paper_2310_04610_b200 as E

    q, k, v, do, b1, b2 = make_inputs(1, 2, 64, 2, 32)
    t = lambda a: torch.tensor(a, dtype=torch.bfloat16, device="cuda")
    o, lse = E.evoformer_attention_forward(t(q), t(k), t(v), t(b1), t(b2))
    assert E.resolved_path(t(q), t(b1), t(b2)) == "tcgen05"
    assert E.last_launch_count() == 1  # K1 alone
    E.evoformer_attention_backward(t(do), t(q), t(k), t(v), o, lse, t(b1), t(b2))
    assert E.last_launch_count() == 3  # preamble, K3, dQ conversion


def test_validation_errors_map_to_taxonomy():
    import paper_2310_04610_b200 as E

    q = torch.zeros(1, 2, 8, 2, 32, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(E.ValidationError):
        E.evoformer_attention_forward(q, q, q[..., :16].contiguous())
    with pytest.raises(E.ValidationError):
        E.evoformer_attention_forward(q, q, q, bias2=torch.zeros(1, 1, 2, 8, 7, dtype=torch.bfloat16, device="cuda"))
    with pytest.raises(E.NumericError):
        E.evoformer_attention_forward(q, q, q, scale=float("nan"))


def _bwd_launches(shape, dtype="bf16"):
    import paper_2310_04610_b200 as E

    q, k, v, do, b1, b2 = make_inputs(*shape, dtype=dtype, seed=5)
    t = lambda a: torch.tensor(a, dtype=TD[dtype], device="cuda")
    o, lse = E.evoformer_attention_forward(t(q), t(k), t(v), t(b1), t(b2))
    E.evoformer_attention_backward(t(do), t(q), t(k), t(v), o, lse, t(b1), t(b2))
    torch.cuda.synchronize()
    return E.last_launch_count()


@pytest.mark.parametrize("shape", [(1, 2, 640, 2, 32), (1, 1, 904, 1, 32)])
def test_tc_backward_query_chunks(shape):
    # L > 384: the tcgen05 backward splits the query axis into chunks of 3 tiles (the chunk's dBias2
    # strip fits in TMEM) and reduces dK/dV over the chunks in fp32; 904 also has ragged last tiles
    check(shape, "bf16")
    assert _bwd_launches(shape) == 5  # prep, main, dQ/dK/dV conversions: the chunked tcgen05 path ran


def test_tc_backward_d16_and_f16():
    check((1, 3, 96, 2, 16), "bf16")
    check((1, 3, 96, 2, 32), "f16")
    assert _bwd_launches((1, 3, 96, 2, 32), "f16") == 3  # prep, main, dQ conversion (tcgen05)


def test_tc_backward_many_rows_per_cta():
    # rows well beyond one per SM: persistent walk over units and row ranges, strip flushes per unit
    check((1, 300, 128, 1, 32), "bf16")


@pytest.mark.parametrize("shape,dtype", [((1, 4, 384, 2, 32), "bf16"), ((2, 2, 200, 2, 32), "bf16"),
                                         ((1, 2, 640, 2, 32), "bf16"), ((1, 3, 200, 2, 16), "f16")])
def test_tc_backward_dbias1(shape, dtype):
    # the mask-bias gradient on the tcgen05 path: column sums of dS from an extra UMMA against a ones
    # block (L = 384 and 640 run in chunks of 2 query tiles to free the TMEM columns)
    check(shape, dtype, need_dbias1=True)


def test_tc_backward_dbias1_stays_on_tcgen05():
    import paper_2310_04610_b200 as E

    q, k, v, do, b1, b2 = make_inputs(1, 2, 384, 2, 32, seed=3)
    t = lambda a: torch.tensor(a, dtype=torch.bfloat16, device="cuda")
    o, lse = E.evoformer_attention_forward(t(q), t(k), t(v), t(b1), t(b2))
    E.evoformer_attention_backward(t(do), t(q), t(k), t(v), o, lse, t(b1), t(b2), need_dbias1=True)
    torch.cuda.synchronize()
    # prep, main (2 query chunks), dQ / dK / dV conversions: the chunked tcgen05 path, not SIMT
    assert E.last_launch_count() == 5


@pytest.mark.parametrize("shape,need_dbias1", [((1, 2, 1024, 2, 32), False), ((1, 2, 640, 2, 32), True),
                                               ((2, 2, 520, 1, 16), False)])
def test_tc_backward_msa_col_unchunked(shape, need_dbias1):
    # MSA column attention (bias-free plus mask, the attended axis is N_seq): without a pair bias
    # there is no dBias2 strip, so the tcgen05 backward takes the whole query axis in one chunk
    check(shape, "bf16", bias2=False, need_dbias1=need_dbias1)
    q, k, v, do, b1, _ = make_inputs(*shape, dtype="bf16", bias2=False, seed=5)
    import paper_2310_04610_b200 as E

    t = lambda a: torch.tensor(a, dtype=torch.bfloat16, device="cuda")
    o, lse = E.evoformer_attention_forward(t(q), t(k), t(v), t(b1))
    E.evoformer_attention_backward(t(do), t(q), t(k), t(v), o, lse, t(b1), None, need_dbias1=need_dbias1)
    torch.cuda.synchronize()
    assert E.last_launch_count() == 3  # prep, main, dQ conversion: no dK/dV chunk reduction


def test_dbias1_request_needs_descriptor_flag():
    # the workspace is sized for the dBias1 path only when desc.need_dbias1 says so: a dbias1
    # request without it is a ValidationError at the C-ABI, before any launch
    import paper_2310_04610_b200 as E
    from paper_2310_04610_b200 import _native as N
    from paper_2310_04610_b200.evoformer_attention import make_desc

    q, k, v, do, b1, b2 = make_inputs(1, 2, 384, 2, 32, seed=9)
    t = lambda a: torch.tensor(a, dtype=torch.bfloat16, device="cuda")
    tq, tk, tv, tdo, tb1, tb2 = map(t, (q, k, v, do, b1, b2))
    o, lse = E.evoformer_attention_forward(tq, tk, tv, tb1, tb2)
    d = make_desc(tq, tb1, tb2, None)
    lib = N.load()
    wsb = lib.evo_attn_bwd_workspace_size(d)
    ws = torch.empty(wsb, device="cuda", dtype=torch.uint8)
    g = [torch.empty_like(tq) for _ in range(3)]
    db1 = torch.empty(tb1.shape, device="cuda", dtype=torch.float32)
    db2 = torch.empty(tb2.shape, device="cuda", dtype=torch.float32)
    p = lambda x: x.data_ptr()
    st = lib.evo_attn_bwd(d, p(tdo), p(tq), p(tk), p(tv), p(tb1), p(tb2), p(o), p(lse), *map(p, g), p(db1),
                          p(db2), 0, p(ws), wsb, torch.cuda.current_stream().cuda_stream)
    assert st == N.EVO_ERR_VALIDATION
    assert "need_dbias1" in lib.evo_attn_last_error().decode()


def test_fwd_streamed_bias_flat_split_segments():
    # L = 1024 streams the pair bias through a 3-slot ring shared by the warpgroups; H = 5 makes the
    # grid a flat item split, so CTAs cross segment boundaries with partial row groups (a warpgroup
    # with no row keeps the ring in step). Regression: a lagging warp of such a warpgroup missed a
    # ring phase and hung (C5); repeated launches give the race a chance.
    import paper_2310_04610_b200 as E
    from tests.util import O

    Bo, Nr, L, H, D = 1, 24, 1024, 5, 32
    q, k, v, _, b1, b2 = make_inputs(Bo, Nr, L, H, D, dtype="bf16", seed=13)
    t = lambda a: torch.tensor(a, dtype=torch.bfloat16, device="cuda")
    tq, tk, tv, tb1, tb2 = map(t, (q, k, v, b1, b2))
    for _ in range(5):
        o, lse = E.evoformer_attention_forward(tq, tk, tv, tb1, tb2)
    torch.cuda.synchronize()
    p = O.Problem(Bo * Nr, L, H, D, fmt=O.F32, Bo=Bo)
    r = lambda a: a.reshape(-1).astype(np.float64)
    wo, wl = O.forward(p, r(q), r(k), r(v), r(b1), r(b2))
    assert nmax_err(o.float().cpu().numpy(), wo.reshape(q.shape)) <= 1e-2
    assert nmax_err(lse.cpu().numpy(), wl.transpose(1, 0, 2)) <= 1e-2
