"""Shared test helpers: seeded OpenFold-shaped inputs and the parity metric.

Input recipe follows SURVEY §8(d): U[-1,1) in fp32, rounded ONCE to the
problem dtype (RNE), the identical values handed to the oracle in float64;
bias1 (mask) in {0, -1e9} at a 10% rate with key 0 never masked.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def make_inputs(Bo, Nr, L, H, D, dtype="bf16", bias1=True, bias2=True, seed=0, mask_rate=0.1):
    rng = np.random.default_rng(seed)
    shape = (Bo, Nr, L, H, D)
    f = lambda s: rng.uniform(-1, 1, s).astype(np.float32)
    q, k, v, do = f(shape), f(shape), f(shape), f(shape)
    b2 = f((Bo, 1, H, L, L)) if bias2 else None
    b1 = None
    if bias1:
        m = rng.uniform(0, 1, (Bo, Nr, 1, 1, L)) < mask_rate
        m[..., 0] = False
        neg = -3.0e4 if dtype == "f16" else -1e9  # -1e9 overflows fp16
        b1 = np.where(m, np.float32(neg), np.float32(0)).astype(np.float32)
    rnd = (lambda a: a) if dtype == "f32" else (lambda a: None if a is None else O.round_to(a, dtype).astype(np.float32))
    return tuple(None if a is None else rnd(a) for a in (q, k, v, do, b1, b2))


def oracle_fwd_bwd(q, k, v, do, b1, b2, scale=None, need_dbias1=False, tile=(64, 64, 1), fmt=None):
    """Oracle (F32 semantics of attention_tiled.cpp) on identically-rounded inputs.
    Returns O [Bo,N,L,H,D], LSE [B,H,L], dQ, dK, dV, dB1 [Bo,N,1,1,L], dB2 [Bo,1,H,L,L]."""
    Bo, Nr, L, H, D = q.shape
    B = Bo * Nr
    p = O.Problem(B, L, H, D, fmt=O.F32 if fmt is None else fmt, Bo=Bo, scale=scale, tile_q=tile[0], tile_k=tile[1],
                  tile_b=tile[2])
    r = lambda a: None if a is None else a.reshape(-1).astype(np.float64)
    o, lse = O.forward(p, r(q), r(k), r(v), r(b1), r(b2))
    dq, dk, dv, db1, db2 = O.backward(p, r(q), r(k), r(v), o, lse, r(do), r(b1), r(b2),
                                      want_dbias1=need_dbias1)
    sh = q.shape
    return (o.reshape(sh), lse.transpose(1, 0, 2), dq.reshape(sh), dk.reshape(sh), dv.reshape(sh),
            None if db1 is None else db1.reshape(Bo, Nr, 1, 1, L),
            None if db2 is None else db2.reshape(Bo, 1, H, L, L))


def nmax_err(got, want) -> float:
    """Normalized max-abs error max|got-want| / max|want|."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(np.abs(want).max(), 1e-30)
    return float(np.abs(got - want).max() / scale)


def ref_rel_err(got, want) -> float:
    """The reference harness's floored max relative error (run.cpp:309-322)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    floor = max(1e-3 * np.abs(want).max(), 1e-8)
    den = np.maximum(np.maximum(np.abs(got), np.abs(want)), floor)
    return float((np.abs(got - want) / den).max())


TOL = {"f32": 1e-4, "bf16": 1e-2, "f16": 1e-2}


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, dtype=np.float64)))


def oracle_fwd_bwd_gated(q, k, v, do_g, b1, b2, gate, scale=None, need_dbias1=False, fmt=None):
    """The fused output gate (OpenFold: o_g = sigmoid(G) * O) composed around the oracle: the oracle
    computes O and the attention backward with dO = do_g * sigmoid(G); dG = do_g * O * s (1 - s).
    Returns (o_g, LSE, dQ, dK, dV, dG, dB1, dB2)."""
    s = sigmoid(gate)
    do = np.asarray(do_g, np.float64) * s
    o, lse, dq, dk, dv, db1, db2 = oracle_fwd_bwd(q, k, v, do, b1, b2, scale=scale, need_dbias1=need_dbias1, fmt=fmt)
    dg = np.asarray(do_g, np.float64) * o * s * (1.0 - s)
    return o * s, lse, dq, dk, dv, dg, db1, db2
