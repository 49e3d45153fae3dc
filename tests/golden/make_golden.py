"""Generate golden fixtures from the REFERENCE ITSELF (oracle/_ref, compiled from
/root/reference sources) — run in the build container, where /root/reference
exists:  python tests/golden/make_golden.py
The .npz files are committed; tests/test_oracle.py::test_golden_fixture checks
the C restatement against them anywhere (including the GPU box).
"""
import json
import zlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402

CASES = [
    # name, variant, B, L, H, D, fmt, tile
    ("msa_row_f32_b2_l20", "msa_row", 2, 20, 2, 8, O.F32, (8, 8, 1)),
    ("tri_start_f64_l12", "tri_start", 12, 12, 2, 4, O.F64, (4, 8, 1)),
    ("msa_col_f32_l17", "msa_col", 3, 17, 1, 4, O.F32, (64, 64, 1)),
    ("msa_row_f32_l33_d32", "msa_row", 2, 33, 1, 32, O.F32, (16, 16, 2)),
]


def main():
    for name, variant, B, L, H, D, fmt, tile in CASES:
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        g = lambda s: O.round_to(rng.uniform(-1, 1, s), "f32")
        q, k, v, do = (g((B, L, H, D)) for _ in range(4))
        bias = g((H, L, L)) if variant != "msa_col" else None
        o, lse, dq, dk, dv, db, peak = O.ref_tiled(variant, fmt, q, k, v, bias, do, tile=tile)
        meta = dict(variant=variant, B=B, L=L, H=H, D=D, fmt=fmt, tile=list(tile), ledger_peak=peak,
                    source="oracle/_ref/libevomem_ref.so (attn_forward_tiled + attn_backward_tiled)")
        arrs = dict(q=q, k=k, v=v, dout=do, o=o, lse=lse, dq=dq, dk=dk, dv=dv, meta=json.dumps(meta))
        if bias is not None:
            arrs.update(bias=bias, dbias=db)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrs)
        print("wrote", name)


if __name__ == "__main__":
    main()
