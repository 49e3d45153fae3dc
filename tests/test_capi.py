"""The C-ABI library loads and exports every symbol include/evoattn.h declares;
validation paths map to the reference error taxonomy (CPU only: no kernel runs)."""
import ctypes as C
import math
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "evoattn.h")).read()
    return sorted(set(re.findall(r"\b(evo_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("evo_attn_fwd", "evo_attn_bwd", "evo_attn_fwd_workspace_size",
                 "evo_attn_bwd_workspace_size", "evo_attn_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2310_04610_b200 import _native as N

    lib = N.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(N.EXPORTED) == set(_declared())
    assert lib.evo_attn_version().decode().startswith("evoattn")


def _desc(**kw):
    from paper_2310_04610_b200 import _native as N

    d = dict(Bo=1, N=4, L=64, H=2, D=32, dtype=N.EVO_BF16, scale=1 / math.sqrt(32), has_bias1=1,
             has_bias2=1, dbias_dtype=N.EVO_F32, path=N.EVO_PATH_AUTO)
    d.update(kw)
    return N.Desc(**d)


def test_workspace_sizes():
    from paper_2310_04610_b200 import _native as N

    lib = N.load()
    d = _desc(need_dbias1=1)
    ws = lib.evo_attn_bwd_workspace_size(d)
    # delta (B*H*L f32) + dbias2 fp32 (H*L*L) + dbias1 (B*L) at least
    assert ws >= 4 * (4 * 2 * 64 + 2 * 64 * 64 + 4 * 64)
    assert lib.evo_attn_bwd_workspace_size(_desc(L=0)) == 0
    # the dBias1 path (query chunks of 2 tiles, fp32 dK/dV) is only budgeted when asked for: at
    # L = 384 it adds two fp32 [B, L, H, D] accumulators
    acc = 4 * 4 * 384 * 2 * 32
    plain = lib.evo_attn_bwd_workspace_size(_desc(L=384))
    with_db1 = lib.evo_attn_bwd_workspace_size(_desc(L=384, need_dbias1=1))
    assert with_db1 - plain >= 2 * acc


def test_status_codes_without_gpu():
    from paper_2310_04610_b200 import _native as N

    lib = N.load()
    st = lib.evo_attn_fwd(None, 1, 1, 1, None, None, 1, 1, None, 0, None)
    assert st == N.EVO_ERR_USAGE
    st = lib.evo_attn_fwd(_desc(L=0), 1, 1, 1, 1, 1, 1, 1, None, 0, None)
    assert st == N.EVO_ERR_VALIDATION and "extents" in lib.evo_attn_last_error().decode()
    st = lib.evo_attn_fwd(_desc(scale=float("inf")), 1, 1, 1, 1, 1, 1, 1, None, 0, None)
    assert st == N.EVO_ERR_NUMERIC
    st = lib.evo_attn_fwd(_desc(), 1, 1, 1, None, 1, 1, 1, None, 0, None)  # bias1 missing
    assert st == N.EVO_ERR_VALIDATION
    with pytest.raises(N.ValidationError):
        N.check(N.EVO_ERR_VALIDATION)
    st = lib.evo_attn_bwd(_desc(dbias_dtype=N.EVO_BF16), 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, None, 1,
                          1, 1, 10**9, None)
    assert st == N.EVO_ERR_VALIDATION  # accumulate requires fp32 dbias
    # raw (axes-swapped) layout: one outer batch only, forward only
    st = lib.evo_attn_fwd(_desc(Bo=2, axes_swapped=1), 1, 1, 1, 1, 1, 1, 1, None, 0, None)
    assert st == N.EVO_ERR_VALIDATION and "Bo == 1" in lib.evo_attn_last_error().decode()
    st = lib.evo_attn_fwd(_desc(axes_swapped=2), 1, 1, 1, 1, 1, 1, 1, None, 0, None)
    assert st == N.EVO_ERR_VALIDATION
    st = lib.evo_attn_bwd(_desc(Bo=2, axes_swapped=1), 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, None, 1,
                          0, 1, 10**9, None)
    assert st == N.EVO_ERR_VALIDATION


def test_simt_path_for_fp32():
    from paper_2310_04610_b200 import _native as N

    lib = N.load()
    assert lib.evo_attn_resolved_path(_desc(dtype=N.EVO_F32, dbias_dtype=N.EVO_F32)) == N.EVO_PATH_SIMT


def _pb_desc(**kw):
    from paper_2310_04610_b200 import _native as N

    d = dict(Bo=1, L=64, C=128, H=8, dtype=N.EVO_BF16, dbias_dtype=N.EVO_F32, eps=1e-5)
    d.update(kw)
    return N.PairBiasDesc(**d)


@pytest.mark.parametrize("kw,status", [
    (dict(C=48), "UNSUPPORTED"),          # c_z not a multiple of 32
    (dict(C=512), "UNSUPPORTED"),         # beyond the 256-channel envelope
    (dict(H=17), "UNSUPPORTED"),
    (dict(dtype=0), "VALIDATION"),        # z must be 16-bit
    (dict(dbias_dtype=2), "VALIDATION"),  # f16 dBias with bf16 z
    (dict(eps=0.0), "NUMERIC"),
    (dict(L=0), "VALIDATION"),
])
def test_pair_bias_descriptor_validation(kw, status):
    """The pair-bias projection's descriptor checks run before any device work (CPU only)."""
    from paper_2310_04610_b200 import _native as N

    lib = N.load()
    d = _pb_desc(**kw)
    st = lib.evo_pair_bias_fwd(C.byref(d), 1, 1, 1, 1, 1, None)
    assert st == getattr(N, f"EVO_ERR_{status}"), lib.evo_attn_last_error()
    assert lib.evo_pair_bias_bwd_workspace_size(C.byref(d)) == 0
    assert lib.evo_pair_bias_fwd(None, 1, 1, 1, 1, 1, None) == N.EVO_ERR_USAGE


def test_pair_bias_workspace_and_null_pointers():
    from paper_2310_04610_b200 import _native as N

    lib = N.load()
    d = _pb_desc()
    assert lib.evo_pair_bias_bwd_workspace_size(C.byref(d)) > 0
    assert lib.evo_pair_bias_fwd(C.byref(d), None, 1, 1, 1, 1, None) == N.EVO_ERR_VALIDATION
    ws = lib.evo_pair_bias_bwd_workspace_size(C.byref(d))
    st = lib.evo_pair_bias_bwd(C.byref(d), 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, ws - 1, None)
    assert st == N.EVO_ERR_VALIDATION  # workspace smaller than required
