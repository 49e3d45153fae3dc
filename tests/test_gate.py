"""The fused OpenFold output gate (not in the reference):
o_g = sigmoid(G) * attention. CPU: the oracle composition (tests/util.oracle_fwd_bwd_gated) is pinned by
a float64 finite-difference gradcheck of every gradient including dG. GPU: the fused kernels (the gate
in the forward epilogue, the gate backward in the backward preamble) against it."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.util import TOL, make_inputs, nmax_err, oracle_fwd_bwd, oracle_fwd_bwd_gated, sigmoid


def _loss(q, k, v, b1, b2, g, w):
    o = oracle_fwd_bwd(q, k, v, np.zeros_like(q), b1, b2, fmt=O.F64)[0]
    return float((sigmoid(g) * o * w).sum())


def test_gate_composition_finite_difference_gradcheck():
    # float64 oracle, central differences (the reference's gradcheck pattern, run.cpp:279-322)
    rng = np.random.default_rng(3)
    q, k, v, w, b1, b2 = make_inputs(1, 2, 5, 1, 3, dtype="f32", seed=4)
    q, k, v, w = (a.astype(np.float64) for a in (q, k, v, w))
    b1, b2 = b1.astype(np.float64), b2.astype(np.float64)
    b1[b1 < -1] = -3.0  # finite mask values keep the FD well conditioned
    g = rng.uniform(-2, 2, q.shape)
    og, _, dq, dk, dv, dg, db1, db2 = oracle_fwd_bwd_gated(q, k, v, w, b1, b2, g, need_dbias1=True, fmt=O.F64)
    h = 1e-6
    for name, x, grad in (("q", q, dq), ("k", k, dk), ("v", v, dv), ("gate", g, dg), ("bias2", b2, db2),
                          ("bias1", b1, db1)):
        fd = np.zeros_like(x)
        it = np.nditer(x, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            orig = x[i]
            x[i] = orig + h
            fp = _loss(q, k, v, b1, b2, g, w)
            x[i] = orig - h
            fm = _loss(q, k, v, b1, b2, g, w)
            x[i] = orig
            fd[i] = (fp - fm) / (2 * h)
        err = np.abs(fd - grad).max() / max(np.abs(fd).max(), 1e-12)
        assert err < 1e-6, (name, err)


def _gpu(q, k, v, do, b1, b2, g, dtype, path="auto"):
    import paper_2310_04610_b200 as E

    td = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[dtype]
    t = lambda a: None if a is None else torch.tensor(a, dtype=td, device="cuda")
    tq, tk, tv, tdo, tb1, tb2, tg = map(t, (q, k, v, do, b1, b2, g))
    o, lse = E.evoformer_attention_forward_gated(tq, tk, tv, tg, tb1, tb2, path=path)
    dq, dk, dv, dg, db1, db2 = E.evoformer_attention_backward_gated(tdo, tq, tk, tv, tg, o, lse, tb1, tb2, path=path)
    torch.cuda.synchronize()
    return [x.float().cpu().numpy() for x in (o, lse, dq, dk, dv, dg, db2)]


@pytest.mark.gpu
@pytest.mark.parametrize("shape,dtype,path", [((1, 4, 128, 2, 32), "bf16", "auto"), ((1, 3, 384, 4, 32), "bf16", "auto"),
                                              ((1, 4, 130, 2, 32), "bf16", "auto"), ((1, 3, 96, 2, 16), "f16", "auto"),
                                              ((1, 2, 64, 2, 32), "f32", "auto"), ((1, 4, 128, 2, 32), "bf16", "simt")])
def test_gated_operator_parity(shape, dtype, path):
    q, k, v, do, b1, b2 = make_inputs(*shape, dtype=dtype, seed=7)
    g = make_inputs(*shape, dtype=dtype, seed=8, bias1=False, bias2=False)[0] * 3.0
    if dtype != "f32":
        g = O.round_to(g, dtype).astype(np.float32)
    got = _gpu(q, k, v, do, b1, b2, g, dtype, path)
    og, lse, dq, dk, dv, dg, _, db2 = oracle_fwd_bwd_gated(q, k, v, do, b1, b2, g)
    want = [og, lse, dq, dk, dv, dg, db2]
    tol = TOL[dtype]
    for name, a, w in zip(["O_gated", "LSE", "dQ", "dK", "dV", "dGate", "dBias2"], got, want):
        assert np.isfinite(a).all(), name
        assert nmax_err(a, w) <= tol, (name, nmax_err(a, w))


@pytest.mark.gpu
def test_ds4sci_with_gate_autograd():
    import paper_2310_04610_b200 as E

    q, k, v, do, b1, b2 = make_inputs(1, 4, 128, 2, 32, dtype="bf16", seed=9)
    g = O.round_to(make_inputs(1, 4, 128, 2, 32, dtype="bf16", seed=10, bias1=False, bias2=False)[0] * 3.0,
                   "bf16").astype(np.float32)
    t = lambda a: torch.tensor(a, dtype=torch.bfloat16, device="cuda").requires_grad_(True)
    tq, tk, tv, tb2, tg = map(t, (q, k, v, b2, g))
    tb1 = torch.tensor(b1, dtype=torch.bfloat16, device="cuda")
    out = E.DS4Sci_EvoformerAttention(tq, tk, tv, [tb1, tb2], gate=tg)
    out.backward(torch.tensor(do, dtype=torch.bfloat16, device="cuda"))
    og, _, dq, dk, dv, dg, _, db2 = oracle_fwd_bwd_gated(q, k, v, do, b1, b2, g)
    for name, a, w in (("O_gated", out.detach(), og), ("dQ", tq.grad, dq), ("dK", tk.grad, dk), ("dV", tv.grad, dv),
                       ("dGate", tg.grad, dg), ("dBias2", tb2.grad, db2)):
        assert nmax_err(a.float().cpu().numpy(), w) <= 1.5e-2, name
