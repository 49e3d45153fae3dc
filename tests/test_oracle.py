"""Pin the oracle (C restatement) before trusting it (CPU only).

1. Bit-for-bit against the reference library itself (oracle/_ref, compiled from
   /root/reference sources) on the reference's own harness shapes.
2. Against committed golden fixtures (tests/golden/, made by
   tests/golden/make_golden.py from oracle/_ref) so the check runs where
   /root/reference is absent.
3. The SPEC worked examples and a finite-difference
   gradcheck (run.cpp:279-357 pattern) that also pins the bias1 extension.
"""
import json
import math
import os
import zlib

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand(rng, shape):
    return O.round_to(rng.uniform(-1, 1, shape), "f32")


CASES = [  # (variant, B, L, H, D, fmt, tile, deterministic)
    ("msa_row", 4, 130, 2, 8, O.F32, (64, 64, 1), True),   # attn-bench default rows (run.cpp:137-157)
    ("msa_col", 4, 130, 2, 8, O.F32, (64, 64, 1), True),
    ("tri_start", 30, 30, 2, 8, O.F32, (16, 8, 1), True),
    ("msa_row", 3, 70, 2, 4, O.F64, (64, 64, 1), True),
    ("msa_row", 3, 70, 2, 4, O.F32, (16, 32, 2), False),   # tile_b > 1, descending batch order
    ("msa_row", 2, 16, 2, 4, O.F64, (8, 8, 1), True),      # gradcheck shape (run.cpp:341)
]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("case", CASES)
def test_bit_exact_vs_reference(case):
    variant, B, L, H, D, fmt, tile, det = case
    rng = np.random.default_rng(zlib.crc32(repr(case).encode()))
    q, k, v, do = (_rand(rng, (B, L, H, D)) for _ in range(4))
    bias = _rand(rng, (H, L, L)) if variant != "msa_col" else None
    ro, rlse, rdq, rdk, rdv, rdb, _ = O.ref_tiled(variant, fmt, q, k, v, bias, do, tile=tile,
                                                  deterministic=det)
    p = O.Problem(B, L, H, D, fmt=fmt, tile_q=tile[0], tile_k=tile[1], tile_b=tile[2],
                  deterministic=det)
    o, lse = O.forward(p, q, k, v, None, bias)
    dq, dk, dv, _, db = O.backward(p, q, k, v, o, lse, do, None, bias)
    for got, want in ((o, ro), (lse, rlse), (dq, rdq), (dk, rdk), (dv, rdv)):
        assert np.array_equal(got, want)
    if bias is not None:
        assert np.array_equal(db[0], rdb)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_bias1_zero_is_bit_identical_to_reference():
    rng = np.random.default_rng(5)
    B, L, H, D = 3, 40, 2, 8
    q, k, v, do = (_rand(rng, (B, L, H, D)) for _ in range(4))
    bias = _rand(rng, (H, L, L))
    ro, rlse, rdq, rdk, rdv, rdb, _ = O.ref_tiled("msa_row", O.F32, q, k, v, bias, do)
    p = O.Problem(B, L, H, D)
    z = np.zeros((B, L))
    o, lse = O.forward(p, q, k, v, z, bias)
    dq, dk, dv, _, db = O.backward(p, q, k, v, o, lse, do, z, bias)
    assert np.array_equal(o, ro) and np.array_equal(dq, rdq) and np.array_equal(db[0], rdb)


def _golden_files():
    if not os.path.isdir(GOLDEN):
        return []
    return sorted(f for f in os.listdir(GOLDEN) if f.endswith(".npz"))


@pytest.mark.parametrize("name", _golden_files())
def test_golden_fixture(name):
    z = np.load(os.path.join(GOLDEN, name))
    meta = json.loads(str(z["meta"]))
    B, L, H, D = meta["B"], meta["L"], meta["H"], meta["D"]
    p = O.Problem(B, L, H, D, fmt=meta["fmt"], tile_q=meta["tile"][0], tile_k=meta["tile"][1],
                  tile_b=meta["tile"][2])
    bias = z["bias"] if "bias" in z.files else None
    o, lse = O.forward(p, z["q"], z["k"], z["v"], None, bias)
    dq, dk, dv, _, db = O.backward(p, z["q"], z["k"], z["v"], o, lse, z["dout"], None, bias)
    assert np.array_equal(o, z["o"]) and np.array_equal(lse, z["lse"])
    assert np.array_equal(dq, z["dq"]) and np.array_equal(dk, z["dk"]) and np.array_equal(dv, z["dv"])
    if bias is not None:
        assert np.array_equal(db[0], z["dbias"])


def test_spec_hand_example():
    # B=1,L=2,H=1,D=1, scale=1, Q=[1,0], K=[1,2], V=[10,20] -> O[0]=(10+20e)/(1+e)
    p = O.Problem(1, 2, 1, 1, fmt=O.F64, scale=1.0)
    q = np.array([1.0, 0.0]).reshape(1, 2, 1, 1)
    k = np.array([1.0, 2.0]).reshape(1, 2, 1, 1)
    v = np.array([10.0, 20.0]).reshape(1, 2, 1, 1)
    o, _ = O.forward(p, q, k, v)
    assert abs(o.ravel()[0] - (10 + 20 * math.e) / (1 + math.e)) < 1e-12
    assert abs(o.ravel()[0] - 17.310585786300) < 1e-9


def test_spec_trivial_cases():
    rng = np.random.default_rng(1)
    B, L, H, D = 2, 5, 2, 4
    # L = 1 => O = V
    p1 = O.Problem(B, 1, H, D, fmt=O.F64)
    q, k, v = (rng.uniform(-1, 1, (B, 1, H, D)) for _ in range(3))
    o, _ = O.forward(p1, q, k, v, None, rng.uniform(-1, 1, (1, H, 1, 1)))
    assert np.array_equal(o, v)
    # zero Q and bias => uniform P => O = mean_j V
    p = O.Problem(B, L, H, D, fmt=O.F64)
    v = rng.uniform(-1, 1, (B, L, H, D))
    o, _ = O.forward(p, np.zeros((B, L, H, D)), rng.uniform(-1, 1, (B, L, H, D)), v, None,
                     np.zeros((1, H, L, L)))
    assert np.allclose(o, np.broadcast_to(v.mean(axis=1, keepdims=True), o.shape), atol=1e-14)
    # dO = 0 => all gradients zero
    q, k = rng.uniform(-1, 1, (B, L, H, D)), rng.uniform(-1, 1, (B, L, H, D))
    bias = rng.uniform(-1, 1, (1, H, L, L))
    o, lse = O.forward(p, q, k, v, None, bias)
    g = O.backward(p, q, k, v, o, lse, np.zeros_like(q), None, bias)
    assert all(np.all(x == 0) for x in (g[0], g[1], g[2], g[4]))


def test_lse_rows_normalise():
    # exp(S - logsumexp) sums to 1 per row
    rng = np.random.default_rng(2)
    B, L, H, D = 2, 37, 2, 8
    q, k, v = (rng.uniform(-1, 1, (B, L, H, D)) for _ in range(3))
    b1 = np.where(rng.uniform(size=(B, L)) < 0.2, -1e9, 0.0)
    b1[:, 0] = 0
    b2 = rng.uniform(-1, 1, (1, H, L, L))
    p = O.Problem(B, L, H, D, fmt=O.F64, tile_q=16, tile_k=16)
    _, lse = O.forward(p, q, k, v, b1, b2)
    s = np.einsum("bihd,bjhd->hbij", q, k) / math.sqrt(D) + b1[None, :, None, :] + b2[0][:, None]
    assert np.allclose(np.exp(s - lse[..., None]).sum(-1), 1.0, atol=1e-12)


def _fd_grad(p, inputs, which, dout, h=1e-5):
    base = [x.copy() if x is not None else None for x in inputs]
    tgt = base[which]
    g = np.zeros_like(tgt)
    flat = tgt.reshape(-1)
    for idx in range(flat.size):
        saved = flat[idx]
        flat[idx] = saved + h
        up = (O.forward(p, *base)[0] * dout).sum()
        flat[idx] = saved - h
        down = (O.forward(p, *base)[0] * dout).sum()
        flat[idx] = saved
        g.reshape(-1)[idx] = (up - down) / (2 * h)
    return g


def _rel(got, want):
    fl = max(1e-3 * np.abs(want).max(), 1e-8)
    return float((np.abs(got - want) / np.maximum(np.maximum(np.abs(got), np.abs(want)), fl)).max())


def test_finite_difference_gradcheck_with_bias1():
    # run.cpp:279-357 pattern (F64, h=1e-5, tol 1e-6), extended to bias1 and Bo=2
    rng = np.random.default_rng(3)
    Bo, Nr, L, H, D = 2, 1, 5, 2, 3
    B = Bo * Nr
    p = O.Problem(B, L, H, D, fmt=O.F64, Bo=Bo, tile_q=2, tile_k=3)
    q, k, v = (rng.uniform(-1, 1, (B, L, H, D)) for _ in range(3))
    b1 = rng.uniform(-1, 1, (B, L))
    b2 = rng.uniform(-1, 1, (Bo, H, L, L))
    dout = rng.uniform(-1, 1, (B, L, H, D))
    o, lse = O.forward(p, q, k, v, b1, b2)
    dq, dk, dv, db1, db2 = O.backward(p, q, k, v, o, lse, dout, b1, b2, want_dbias1=True)
    ins = [q, k, v, b1, b2]
    for which, got in enumerate((dq, dk, dv, db1, db2)):
        assert _rel(got, _fd_grad(p, ins, which, dout)) < 1e-6, which


def test_threaded_driver_matches_single():
    rng = np.random.default_rng(4)
    B, L, H, D = 6, 33, 2, 8
    q, k, v, do = (_rand(rng, (B, L, H, D)) for _ in range(4))
    b2 = _rand(rng, (1, H, L, L))
    p = O.Problem(B, L, H, D)
    o, lse = O.forward(p, q, k, v, None, b2)
    dq, dk, dv, _, db2 = O.backward(p, q, k, v, o, lse, do, None, b2)
    to, tlse, tdq, tdk, tdv, tdb2 = O.fwd_bwd_threaded(p, 3, q, k, v, do, None, b2)
    assert np.array_equal(to, o) and np.array_equal(tdq, dq) and np.array_equal(tdv, dv)
    assert np.abs(tdb2 - db2).max() <= 1e-5 * np.abs(db2).max()


def test_validation_status():
    with pytest.raises(O.OracleError) as e:
        O.forward(O.Problem(1, 4, 1, 2, tile_q=0), *(np.zeros((1, 4, 1, 2)),) * 3)
    assert e.value.status == 1
    x = np.zeros((1, 4, 1, 2))
    x[0, 0, 0, 0] = np.nan
    with pytest.raises(O.OracleError) as e:
        O.forward(O.Problem(1, 4, 1, 2), x, x, x)
    assert e.value.status == 2
