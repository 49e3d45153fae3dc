"""ctypes binding of the C-ABI in include/evoattn.h (libevoattn.so, built in-tree).

The product path has no fallback: if the library is missing or fails to load
on a GPU box, every op raises. Device memory and streams come from torch.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

EVO_OK, EVO_ERR_VALIDATION, EVO_ERR_NUMERIC, EVO_ERR_USAGE, EVO_ERR_CUDA, EVO_ERR_UNSUPPORTED = range(6)
EVO_F32, EVO_BF16, EVO_F16 = 0, 1, 2
EVO_PATH_AUTO, EVO_PATH_SIMT, EVO_PATH_TCGEN05 = 0, 1, 2

# Symbols declared in include/evoattn.h (checked by tests/test_capi.py).
EXPORTED = (
    "evo_attn_fwd_workspace_size", "evo_attn_bwd_workspace_size", "evo_attn_fwd", "evo_attn_bwd",
    "evo_attn_resolved_path", "evo_attn_resolved_bwd_path", "evo_attn_last_launch_count", "evo_attn_last_error",
    "evo_attn_version", "evo_random_uniform", "evo_random_mask", "evo_attn_fwd_gated", "evo_attn_bwd_gated",
    "evo_pair_bias_fwd", "evo_pair_bias_bwd_workspace_size", "evo_pair_bias_bwd",
)


class Desc(C.Structure):
    _fields_ = [("Bo", C.c_int64), ("N", C.c_int64), ("L", C.c_int64), ("H", C.c_int64),
                ("D", C.c_int64), ("dtype", C.c_int), ("scale", C.c_double),
                ("has_bias1", C.c_int), ("has_bias2", C.c_int), ("dbias_dtype", C.c_int),
                ("path", C.c_int), ("dbias2_multicast", C.c_void_p), ("need_dbias1", C.c_int),
                ("axes_swapped", C.c_int), ("check_numerics", C.c_int), ("deterministic", C.c_int),
                ("has_gate", C.c_int)]


class PairBiasDesc(C.Structure):
    _fields_ = [("Bo", C.c_int64), ("L", C.c_int64), ("C", C.c_int64), ("H", C.c_int64),
                ("dtype", C.c_int), ("dbias_dtype", C.c_int), ("eps", C.c_float)]


_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libevoattn.so; compile it first when absent and nvcc exists."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_build.LIB):
        if not build_if_missing:
            raise RuntimeError(f"{_build.LIB} is missing: run __graft_entry__.build()")
        _build.build()
    lib = C.CDLL(_build.LIB)
    vp, sz, dp = C.c_void_p, C.c_size_t, C.POINTER(Desc)
    lib.evo_attn_fwd_workspace_size.argtypes = [dp]
    lib.evo_attn_fwd_workspace_size.restype = sz
    lib.evo_attn_bwd_workspace_size.argtypes = [dp]
    lib.evo_attn_bwd_workspace_size.restype = sz
    lib.evo_attn_fwd.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.evo_attn_fwd.restype = C.c_int
    lib.evo_attn_bwd.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int,
                                 vp, sz, vp]
    lib.evo_attn_bwd.restype = C.c_int
    lib.evo_attn_resolved_path.argtypes = [dp]
    lib.evo_attn_resolved_path.restype = C.c_int
    if hasattr(lib, "evo_attn_resolved_bwd_path"):
        lib.evo_attn_resolved_bwd_path.argtypes = [dp]
        lib.evo_attn_resolved_bwd_path.restype = C.c_int
    lib.evo_attn_last_launch_count.restype = C.c_int
    lib.evo_attn_last_error.restype = C.c_char_p
    lib.evo_attn_version.restype = C.c_char_p
    if hasattr(lib, "evo_attn_fwd_gated"):
        lib.evo_attn_fwd_gated.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        lib.evo_attn_fwd_gated.restype = C.c_int
        lib.evo_attn_bwd_gated.argtypes = [dp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_int,
                                           vp, sz, vp]
        lib.evo_attn_bwd_gated.restype = C.c_int
    if hasattr(lib, "evo_pair_bias_fwd"):
        pd = C.POINTER(PairBiasDesc)
        lib.evo_pair_bias_fwd.argtypes = [pd, vp, vp, vp, vp, vp, vp]
        lib.evo_pair_bias_fwd.restype = C.c_int
        lib.evo_pair_bias_bwd_workspace_size.argtypes = [pd]
        lib.evo_pair_bias_bwd_workspace_size.restype = sz
        lib.evo_pair_bias_bwd.argtypes = [pd, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
        lib.evo_pair_bias_bwd.restype = C.c_int
    if not hasattr(lib, "evo_random_uniform"):  # an older A/B variant (tools/ab_time.py)
        _lib = lib
        return lib
    lib.evo_random_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                       C.c_int, vp]
    lib.evo_random_uniform.restype = C.c_int
    lib.evo_random_mask.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                    C.c_double, C.c_int, vp]
    lib.evo_random_mask.restype = C.c_int
    _lib = lib
    return lib


class EvoAttnError(RuntimeError):
    """Base of the error taxonomy (reference errors.hpp:9-36)."""

    status = -1


class ValidationError(EvoAttnError):
    status = EVO_ERR_VALIDATION


class NumericError(EvoAttnError):
    status = EVO_ERR_NUMERIC


class UsageError(EvoAttnError):
    status = EVO_ERR_USAGE


class CudaError(EvoAttnError):
    status = EVO_ERR_CUDA


class UnsupportedError(EvoAttnError):
    status = EVO_ERR_UNSUPPORTED


_ERRORS = {c.status: c for c in (ValidationError, NumericError, UsageError, CudaError, UnsupportedError)}


def check(status: int) -> None:
    if status != EVO_OK:
        msg = load().evo_attn_last_error().decode()
        raise _ERRORS.get(status, EvoAttnError)(msg)
