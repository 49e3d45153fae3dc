"""Triangle-end-node forward at C3 (N_res 384, H 4, D 32, bf16): copy-free raw layout
(variant_forward, axes_swapped strides) vs transpose -> canonical forward -> transpose back.
CUDA events on the current stream, 50 iterations after 5 warm-up."""
import torch

import paper_2310_04610_b200 as E
from paper_2310_04610_b200 import variants as Vr


def timed(fn, it=50):
    for _ in range(5):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


def main():
    L, H, D = 384, 4, 32
    g = torch.Generator(device="cuda").manual_seed(0)
    r = lambda *s: (torch.rand(*s, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    q, k, v = r(L, L, H, D), r(L, L, H, D), r(L, L, H, D)
    bias, mask = r(H, L, L), torch.zeros(L, L, device="cuda", dtype=torch.bfloat16)

    def copy_free():
        return Vr.variant_forward("tri_end", q, k, v, bias, mask)

    def transposed():
        qc, kc, vc = (t.transpose(0, 1).contiguous().unsqueeze(0) for t in (q, k, v))
        o, lse = E.evoformer_attention_forward(qc, kc, vc, mask.reshape(1, L, 1, 1, L),
                                               bias.reshape(1, 1, H, L, L))
        return o[0].transpose(0, 1).contiguous(), lse

    o1, _ = copy_free()
    o2, _ = transposed()
    err = (o1.float() - o2.float()).abs().max().item()
    t1, t2 = timed(copy_free), timed(transposed)
    fl = 4 * L * H * L * L * D
    print(f"tri_end fwd C3: copy-free {t1 * 1e3:.1f} us ({fl / t1 / 1e9:.0f} TFLOP/s), "
          f"transposed {t2 * 1e3:.1f} us ({fl / t2 / 1e9:.0f} TFLOP/s), max |diff| {err:.3g}")

    # fwd+bwd through autograd: raw layout in place vs transposing around the canonical operator
    qg, kg, vg = (t.clone().requires_grad_(True) for t in (q, k, v))
    bg = bias.clone().requires_grad_(True)
    do = r(L, L, H, D)

    def step_raw():
        Vr.variant_attention("tri_end", qg, kg, vg, bg, mask).backward(do)

    def step_transposed():
        qc, kc, vc = (t.transpose(0, 1).contiguous().unsqueeze(0) for t in (qg, kg, vg))
        o = E.DS4Sci_EvoformerAttention(qc, kc, vc, [mask.reshape(1, L, 1, 1, L), bg.reshape(1, 1, H, L, L)])
        o[0].transpose(0, 1).backward(do)

    t3, t4 = timed(step_raw, 20), timed(step_transposed, 20)
    fl = 14 * L * H * L * L * D
    print(f"tri_end fwd+bwd C3: raw layout {t3 * 1e3:.1f} us ({fl / t3 / 1e9:.0f} TFLOP/s), "
          f"transposed {t4 * 1e3:.1f} us ({fl / t4 / 1e9:.0f} TFLOP/s)")


if __name__ == "__main__":
    main()
