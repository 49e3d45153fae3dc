"""The synthetic-input port (csrc/evoattn_inputs.cu, paper_2310_04610_b200/inputs.py) against the
reference's own generator (derived_rng + random_uniform, rng.hpp:41-47, rng.cpp:5-10, compiled
into oracle/_ref) — bit-exact — and the rounding against the reference's known answers
(test_tensor.cpp:122-183). CPU only: the generator is host code."""
import numpy as np
import pytest
import torch

from oracle import oracle as O

from paper_2310_04610_b200 import inputs as I

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _f64(t: torch.Tensor) -> np.ndarray:
    return t.to(torch.float64).numpy()


@needs_ref
@pytest.mark.parametrize("fmt", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("seed,stream,skip", [(0, 0, 0), (7, 3, 12345), (2 ** 63 + 5, (1 << 20) + 1, 999)])
def test_port_is_bit_exact_vs_reference(fmt, seed, stream, skip):
    n = 50_000
    want = O.ref_random_uniform(seed, stream, skip, n, fmt)
    got = _f64(I.random_uniform(seed, stream, skip, n, fmt))
    assert np.array_equal(got, want)


@needs_ref
def test_port_wide_range_rounding_matches_reference():
    # values across the whole exponent range incl. bf16/f16 subnormals and f16 overflow to inf
    for fmt in ("bf16", "f16"):
        for lo, hi in ((-1e-40, 1e-40), (-7e-5, 7e-5), (-7e4, 7e4), (-3.5e38, 3.5e38)):
            want = O.ref_random_uniform(3, 1, 0, 20_000, fmt, lo, hi)
            got = _f64(I.random_uniform(3, 1, 0, 20_000, fmt, lo, hi))
            assert np.array_equal(got, want), (fmt, lo, hi)


@needs_ref
def test_random_problem_stream_order_matches_reference():
    # run.cpp:178-195: Q, K, V, then the bias from one stream; dO from stream + 2^20
    B, L, H, D = 3, 10, 2, 4
    p = I.random_problem(1, B, L, H, D, "bf16", seed=11, stream=2, bias1=False)
    n = B * L * H * D
    allv = O.ref_random_uniform(11, 2, 0, 3 * n + H * L * L, "bf16")
    assert np.array_equal(_f64(p.q).ravel(), allv[:n])
    assert np.array_equal(_f64(p.k).ravel(), allv[n:2 * n])
    assert np.array_equal(_f64(p.v).ravel(), allv[2 * n:3 * n])
    assert np.array_equal(_f64(p.bias2).ravel(), allv[3 * n:])
    assert np.array_equal(_f64(p.dout).ravel(), O.ref_random_uniform(11, 2 + (1 << 20), 0, n, "bf16"))


def test_row_shards_draw_the_full_problem_values():
    full = I.random_problem(2, 6, 12, 2, 8, "bf16", seed=5)
    part = I.random_problem(2, 6, 12, 2, 8, "bf16", seed=5, rows=(2, 5))
    for a, b in zip(full[:5], part[:5]):
        assert torch.equal(a[:, 2:5], b)
    assert torch.equal(full.bias2, part.bias2)


def test_mask_recipe():
    m = I.random_mask(7, 0, (0, 400), 64, "bf16").view(400, 64).float()
    assert (m[:, 0] == 0).all()  # key 0 never masked: no fully masked row
    frac = (m < 0).float().mean().item()
    assert 0.07 < frac < 0.13
    assert set(torch.unique(m).tolist()) <= {0.0, float(torch.tensor(-1e9, dtype=torch.bfloat16))}


def test_reference_rounding_known_answers():
    # test_tensor.cpp:122-183: bf16(pi) = 3.140625; ties to even; f16 subnormals; idempotence
    r = lambda x, f: O.round_to(np.array([x]), f)[0]
    assert r(np.pi, "bf16") == 3.140625
    assert r(1.0 + 2 ** -8, "bf16") == 1.0             # tie -> even (mantissa 0)
    assert r(1.0 + 3 * 2 ** -8, "bf16") == 1.0 + 2 ** -6  # tie -> even (round up)
    assert r(2 ** -24, "f16") == 2 ** -24               # smallest f16 subnormal
    assert r(2 ** -26, "f16") == 0.0                    # below half the smallest subnormal
    assert r(1e6, "f16") == np.inf                      # overflow saturates to inf
    x = np.random.default_rng(0).uniform(-4, 4, 100_000)
    for f in ("bf16", "f16"):
        once = O.round_to(x, f)
        assert np.array_equal(O.round_to(once, f), once)
    # the product port rounds identically (draws of U[-1,1) through both)
    got = _f64(I.random_uniform(9, 0, 0, 4096, "bf16"))
    assert np.array_equal(O.round_to(got, "bf16"), got)
