"""ctypes front end of the parity checkers — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module. It wraps
  * libevo_oracle.so        — the C restatement (evo_oracle.c) of
    /root/reference/proj/core/src/attention_tiled.cpp:57-340 plus the bias1
    (mask) extension, and
  * _ref/libevomem_ref.so   — the reference library itself, compiled from its
    own sources by oracle/Makefile (ref_shim.cpp exposes its operator API).
Parity of the restatement is pinned bit-for-bit against the reference in
tests/test_oracle.py and against committed fixtures in tests/golden/.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libevo_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libevomem_ref.so")

F64, F32 = 0, 1
VARIANTS = {"msa_row": 0, "msa_col": 1, "tri_start": 2, "tri_end": 3}

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)


def build(quiet: bool = True) -> None:
    """Compile the checkers (make -C oracle); the reference part only when
    /root/reference is present (this container), else keep the prebuilt .so."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class _Problem(C.Structure):
    _fields_ = [("fmt", C.c_int), ("B", C.c_int64), ("L", C.c_int64), ("H", C.c_int64),
                ("D", C.c_int64), ("Bo", C.c_int64), ("scale", C.c_double),
                ("tile_q", C.c_int64), ("tile_k", C.c_int64), ("tile_b", C.c_int64),
                ("deterministic", C.c_int)]


_lib = None
_ref = None


def _oracle():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        _lib = C.CDLL(ORACLE_SO)
        pp = C.POINTER(_Problem)
        _lib.evo_oracle_forward.restype = C.c_int
        _lib.evo_oracle_forward.argtypes = [pp] + [_dp] * 7
        _lib.evo_oracle_backward.restype = C.c_int
        _lib.evo_oracle_backward.argtypes = [pp] + [_dp] * 13
        _lib.evo_oracle_fwd_bwd_threaded.restype = C.c_int
        _lib.evo_oracle_fwd_bwd_threaded.argtypes = [pp, C.c_int] + [_dp] * 12
        _lib.evo_oracle_round.restype = None
        _lib.evo_oracle_round.argtypes = [_dp, C.c_int64, C.c_int, C.c_int]
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _reflib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise RuntimeError("oracle/_ref/libevomem_ref.so is not built (no /root/reference here)")
        _ref = C.CDLL(REF_SO)
        i, i64, d = C.c_int, C.c_int64, C.c_double
        _ref.evomem_ref_tiled.restype = C.c_int
        _ref.evomem_ref_tiled.argtypes = [i, i, i64, i64, i64, i64, _dp, _dp, _dp, _dp, _dp, d,
                                          i64, i64, i64, i, _dp, _dp, _dp, _dp, _dp, _dp,
                                          C.POINTER(i64)]
        _ref.evomem_ref_naive.restype = C.c_int
        _ref.evomem_ref_naive.argtypes = [i, i, i64, i64, i64, i64, _dp, _dp, _dp, _dp, _dp, d,
                                          _dp, _dp, _dp, _dp, _dp, C.POINTER(i64)]
        _ref.evomem_ref_tiled_threaded_f32.restype = C.c_int
        _ref.evomem_ref_tiled_threaded_f32.argtypes = [i64, i64, i64, i64, _fp, _fp, _fp, _fp,
                                                       _fp, d, i, _fp, _fp, _fp, _fp, _fp]
        _ref.evomem_ref_analytic_bytes.restype = C.c_int64
        _ref.evomem_ref_analytic_bytes.argtypes = [i64, i64, i64, i64, i, i, i, i64, i64, i64]
        _ref.evomem_ref_last_error.restype = C.c_char_p
        _ref.evomem_ref_random_uniform.restype = C.c_int
        _ref.evomem_ref_random_uniform.argtypes = [C.c_uint64, C.c_uint64, i64, i64, i, d, d, _dp]
    return _ref


def _ptr(a: Optional[np.ndarray], kind=_dp):
    if a is None:
        return None
    return a.ctypes.data_as(kind)


def _d(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Problem:
    B: int
    L: int
    H: int
    D: int
    fmt: int = F32
    Bo: int = 1
    scale: Optional[float] = None
    tile_q: int = 64
    tile_k: int = 64
    tile_b: int = 1
    deterministic: bool = True

    def c(self) -> _Problem:
        s = self.scale if self.scale is not None else 1.0 / np.sqrt(self.D)
        return _Problem(self.fmt, self.B, self.L, self.H, self.D, self.Bo, s,
                        self.tile_q, self.tile_k, self.tile_b, int(self.deterministic))


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        super().__init__(f"oracle status {status} {what}")
        self.status = status


def forward(p: Problem, q, k, v, bias1=None, bias2=None):
    """O (B,L,H,D) and LSE (H,B,L) — attn_forward_tiled semantics (+bias1)."""
    q, k, v, bias1, bias2 = map(_d, (q, k, v, bias1, bias2))
    o = np.zeros((p.B, p.L, p.H, p.D))
    lse = np.zeros((p.H, p.B, p.L))
    pc = p.c()
    st = _oracle().evo_oracle_forward(C.byref(pc), _ptr(q), _ptr(k), _ptr(v), _ptr(bias1),
                                      _ptr(bias2), _ptr(o), _ptr(lse))
    if st:
        raise OracleError(st)
    return o, lse


def backward(p: Problem, q, k, v, o, lse, dout, bias1=None, bias2=None, want_dbias1=False):
    q, k, v, o, lse, dout, bias1, bias2 = map(_d, (q, k, v, o, lse, dout, bias1, bias2))
    dq = np.zeros_like(q)
    dk = np.zeros_like(q)
    dv = np.zeros_like(q)
    db1 = np.zeros((p.B, p.L)) if (want_dbias1 and bias1 is not None) else None
    db2 = np.zeros((p.Bo, p.H, p.L, p.L)) if bias2 is not None else None
    pc = p.c()
    st = _oracle().evo_oracle_backward(C.byref(pc), _ptr(q), _ptr(k), _ptr(v), _ptr(bias1),
                                       _ptr(bias2), _ptr(o), _ptr(lse), _ptr(dout), _ptr(dq),
                                       _ptr(dk), _ptr(dv), _ptr(db1), _ptr(db2))
    if st:
        raise OracleError(st)
    return dq, dk, dv, db1, db2


def fwd_bwd_threaded(p: Problem, threads: int, q, k, v, dout, bias1=None, bias2=None):
    q, k, v, dout, bias1, bias2 = map(_d, (q, k, v, dout, bias1, bias2))
    o = np.zeros_like(q)
    lse = np.zeros((p.H, p.B, p.L))
    dq, dk, dv = np.zeros_like(q), np.zeros_like(q), np.zeros_like(q)
    db2 = np.zeros((p.Bo, p.H, p.L, p.L)) if bias2 is not None else None
    pc = p.c()
    st = _oracle().evo_oracle_fwd_bwd_threaded(C.byref(pc), threads, _ptr(q), _ptr(k), _ptr(v),
                                               _ptr(bias1), _ptr(bias2), _ptr(dout), _ptr(o),
                                               _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(db2))
    if st:
        raise OracleError(st)
    return o, lse, dq, dk, dv, db2


def round_to(x: np.ndarray, fmt: str) -> np.ndarray:
    """RNE onto bf16 / f16 / f32 grids exactly like numeric_format.cpp:42-78."""
    mb, eb = {"bf16": (7, 8), "f16": (10, 5), "f32": (23, 8)}[fmt]
    y = np.ascontiguousarray(x, dtype=np.float64).copy()
    _oracle().evo_oracle_round(_ptr(y), C.c_int64(y.size), mb, eb)
    return y


# ----------------------------------------------------------------- reference
def ref_tiled(variant: str, fmt: int, q, k, v, bias, dout, scale=None, tile=(64, 64, 1),
              deterministic=True):
    """The reference's own attn_forward_tiled + attn_backward_tiled."""
    q, k, v, bias, dout = map(_d, (q, k, v, bias, dout))
    B, L, H, D = q.shape
    s = scale if scale is not None else 1.0 / np.sqrt(D)
    o = np.zeros_like(q)
    lse = np.zeros((H, B, L))
    dq, dk, dv = np.zeros_like(q), np.zeros_like(q), np.zeros_like(q)
    db = np.zeros((H, L, L)) if bias is not None else None
    peak = C.c_int64(0)
    lib = _reflib()
    st = lib.evomem_ref_tiled(VARIANTS[variant], fmt, B, L, H, D, _ptr(q), _ptr(k), _ptr(v),
                              _ptr(bias), _ptr(dout), C.c_double(s), tile[0], tile[1], tile[2],
                              int(deterministic), _ptr(o), _ptr(lse), _ptr(dq), _ptr(dk),
                              _ptr(dv), _ptr(db), C.byref(peak))
    if st:
        raise OracleError(st, lib.evomem_ref_last_error().decode())
    return o, lse, dq, dk, dv, db, peak.value


def ref_naive(variant: str, fmt: int, q, k, v, bias, dout, scale=None):
    q, k, v, bias, dout = map(_d, (q, k, v, bias, dout))
    B, L, H, D = q.shape
    s = scale if scale is not None else 1.0 / np.sqrt(D)
    o = np.zeros_like(q)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(q), np.zeros_like(q)
    db = np.zeros((H, L, L)) if bias is not None else None
    peak = C.c_int64(0)
    lib = _reflib()
    st = lib.evomem_ref_naive(VARIANTS[variant], fmt, B, L, H, D, _ptr(q), _ptr(k), _ptr(v),
                              _ptr(bias), _ptr(dout), C.c_double(s), _ptr(o), _ptr(dq), _ptr(dk),
                              _ptr(dv), _ptr(db), C.byref(peak))
    if st:
        raise OracleError(st, lib.evomem_ref_last_error().decode())
    return o, dq, dk, dv, db, peak.value


def ref_threaded_f32(q, k, v, bias, dout, threads: int, scale=None):
    """Reference tiled fwd+bwd in F32 over `threads` row shards (CPU baseline)."""
    f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)
    q, k, v, bias, dout = map(f, (q, k, v, bias, dout))
    B, L, H, D = q.shape
    s = scale if scale is not None else 1.0 / np.sqrt(D)
    o, dq, dk, dv = (np.zeros_like(q) for _ in range(4))
    db = np.zeros((H, L, L), np.float32) if bias is not None else None
    lib = _reflib()
    st = lib.evomem_ref_tiled_threaded_f32(B, L, H, D, _ptr(q, _fp), _ptr(k, _fp), _ptr(v, _fp),
                                           _ptr(bias, _fp), _ptr(dout, _fp), C.c_double(s),
                                           threads, _ptr(o, _fp), _ptr(dq, _fp), _ptr(dk, _fp),
                                           _ptr(dv, _fp), _ptr(db, _fp))
    if st:
        raise OracleError(st, lib.evomem_ref_last_error().decode())
    return o, dq, dk, dv, db


def ref_analytic_bytes(H, B, L, D, bytes_per_elem, tiled, backward, tile=(64, 64), workers=1):
    return int(_reflib().evomem_ref_analytic_bytes(H, B, L, D, bytes_per_elem, int(tiled),
                                                   int(backward), tile[0], tile[1], workers))


def ref_random_uniform(seed: int, stream: int, skip: int, n: int, fmt: str, lo=-1.0, hi=1.0) -> np.ndarray:
    """The reference's derived_rng + random_uniform (rng.hpp:41-47): n values after `skip` draws."""
    out = np.zeros(n)
    f = {"f64": 0, "f32": 1, "bf16": 2, "f16": 3}[fmt]
    lib = _reflib()
    st = lib.evomem_ref_random_uniform(seed, stream, skip, n, f, lo, hi, _ptr(out))
    if st:
        raise OracleError(st, lib.evomem_ref_last_error().decode())
    return out
