"""Reference-identical synthetic inputs (host side, not the hot path).

Port of the reference's instance generator so that the bench, the reference arm and the parity
tests see the SAME values:
  random_problem(c, seed, stream)  run.cpp:178-189  Q, K, V, then the pair bias, all from one stream
                                                    derived_rng(seed, stream) (rng.hpp:41-43)
  grad_out                         run.cpp:194-195  from stream + 2^20
  random_uniform                   rng.cpp:5-10     U[-1, 1) rounded to the problem format
The DS4Sci mask bias1 (no reference counterpart) comes from stream + 2^21: per (row, key) one draw,
-1e9 (-3e4 for f16) where the draw < mask_rate, key 0 never masked. The generator itself is C++ in
the native library (csrc/evoattn_inputs.cu; pinned to oracle/_ref in tests/test_inputs.py); each
tensor is drawn on its own host thread (the engine discards the draws of the tensors before it).
"""
from __future__ import annotations

import concurrent.futures as cf
from typing import NamedTuple, Optional, Tuple

import torch

from . import _native as N

_DTYPES = {"f32": (torch.float32, N.EVO_F32), "bf16": (torch.bfloat16, N.EVO_BF16),
           "f16": (torch.float16, N.EVO_F16)}
DOUT_STREAM = 1 << 20
MASK_STREAM = 1 << 21


class Problem(NamedTuple):
    q: torch.Tensor      # [Bo, n_rows, L, H, D]
    k: torch.Tensor
    v: torch.Tensor
    dout: torch.Tensor
    bias1: Optional[torch.Tensor]  # [Bo, n_rows, 1, 1, L]
    bias2: Optional[torch.Tensor]  # [Bo, 1, H, L, L]


def random_uniform(seed: int, stream: int, skip: int, n: int, dtype: str = "bf16", lo: float = -1.0,
                   hi: float = 1.0, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Draws [skip, skip + n) of derived_rng(seed, stream) as random_uniform values (host tensor)."""
    tdt, edt = _DTYPES[dtype]
    if out is None:
        out = torch.empty(n, dtype=tdt)
    assert out.dtype == tdt and out.is_contiguous() and out.numel() == n and not out.is_cuda
    N.check(N.load().evo_random_uniform(seed, stream, skip, n, lo, hi, edt, out.data_ptr()))
    return out


def random_mask(seed: int, stream: int, rows: Tuple[int, int], L: int, dtype: str = "bf16",
                rate: float = 0.1, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    tdt, edt = _DTYPES[dtype]
    lo, hi = rows
    neg = -3.0e4 if dtype == "f16" else -1e9
    if out is None:
        out = torch.empty((hi - lo) * L, dtype=tdt)
    N.check(N.load().evo_random_mask(seed, stream + MASK_STREAM, hi - lo, lo, L, rate, neg, edt, out.data_ptr()))
    return out


def random_problem(Bo: int, Nr: int, L: int, H: int, D: int, dtype: str = "bf16", seed: int = 7,
                   stream: int = 0, rows: Optional[Tuple[int, int]] = None, bias1: bool = True,
                   bias2: bool = True, mask_rate: float = 0.1, pin: bool = False) -> Problem:
    """The reference's random_problem for B = Bo*Nr canonical rows (Q, K, V, bias from one stream in
    that order), its grad_out stream, and the DS4Sci mask. `rows` = (lo, hi) selects rows of every
    outer batch (row shards of a sharded launch draw exactly the full problem's values)."""
    tdt, _ = _DTYPES[dtype]
    lo, hi = rows if rows is not None else (0, Nr)
    n_row = L * H * D
    B = Bo * Nr
    nb = hi - lo
    mk = lambda *s: torch.empty(*s, dtype=tdt, pin_memory=pin)
    q, k, v, do = (mk(Bo, nb, L, H, D) for _ in range(4))
    b2 = mk(Bo, 1, H, L, L) if bias2 else None
    b1 = mk(Bo, nb, 1, 1, L) if bias1 else None
    jobs = []
    for ob in range(Bo):
        first = (ob * Nr + lo) * n_row
        for t, base, st in ((q, 0, stream), (k, B * n_row, stream), (v, 2 * B * n_row, stream),
                            (do, 0, stream + DOUT_STREAM)):
            jobs.append((random_uniform, (seed, st, base + first, nb * n_row, dtype), {"out": t[ob].view(-1)}))
        if b1 is not None:
            jobs.append((random_mask, (seed, stream, (ob * Nr + lo, ob * Nr + hi), L, dtype),
                         {"rate": mask_rate, "out": b1[ob].view(-1)}))
    if b2 is not None:
        jobs.append((random_uniform, (seed, stream, 3 * B * n_row, Bo * H * L * L, dtype), {"out": b2.view(-1)}))
    with cf.ThreadPoolExecutor(max_workers=min(len(jobs), 8)) as ex:
        for f in [ex.submit(fn, *a, **kw) for fn, a, kw in jobs]:
            f.result()
    return Problem(q, k, v, do, b1, b2)
