"""Developer check: forward/backward of every kernel path vs the oracle on a few shapes,
printing normalized max errors (used while bringing up the tcgen05 kernels)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2310_04610_b200 as E
from tests.util import make_inputs, nmax_err, oracle_fwd_bwd

SHAPES = [  # Bo, N, L, H, D, bias1, bias2
    (1, 2, 128, 1, 32, False, False),
    (1, 2, 128, 2, 32, True, True),
    (1, 3, 256, 2, 32, True, True),
    (1, 2, 384, 2, 32, True, True),
    (1, 2, 130, 2, 32, True, True),
    (2, 2, 200, 2, 32, True, True),
    (1, 2, 96, 2, 16, True, True),
    (1, 2, 192, 2, 64, True, True),
    (1, 1, 640, 1, 32, True, True),
    # many rows per CTA (persistent walk, segment boundaries)
    (1, 300, 128, 1, 32, False, False),
    (1, 300, 128, 1, 32, True, True),
    (1, 160, 256, 2, 32, True, True),
    (2, 40, 384, 2, 32, True, True),
]
if "--multi" in sys.argv:
    SHAPES = SHAPES[-4:]

only_fwd = "--fwd" in sys.argv
for shp in SHAPES:
    Bo, Nr, L, H, D, b1on, b2on = shp
    q, k, v, do, b1, b2 = make_inputs(Bo, Nr, L, H, D, dtype="bf16", bias1=b1on, bias2=b2on, seed=3)
    want = oracle_fwd_bwd(q, k, v, do, b1, b2)
    t = lambda a: None if a is None else torch.tensor(a, dtype=torch.bfloat16, device="cuda")
    tq, tk, tv, tdo, tb1, tb2 = map(t, (q, k, v, do, b1, b2))
    for path in ("simt", "tcgen05"):
        try:
            o, lse = E.evoformer_attention_forward(tq, tk, tv, tb1, tb2, path=path)
            torch.cuda.synchronize()
            errs = [nmax_err(o.float().cpu().numpy(), want[0]), nmax_err(lse.cpu().numpy(), want[1])]
            if not only_fwd:
                dq, dk, dv, _, db2 = E.evoformer_attention_backward(tdo, tq, tk, tv, o, lse, tb1, tb2, path=path)
                torch.cuda.synchronize()
                errs += [nmax_err(x.float().cpu().numpy(), w) for x, w in ((dq, want[2]), (dk, want[3]), (dv, want[4]))]
                if db2 is not None:
                    errs.append(nmax_err(db2.cpu().numpy(), want[6]))
            print(shp, path, " ".join(f"{e:.2e}" for e in errs), flush=True)
        except Exception as ex:
            print(shp, path, "ERROR", repr(ex)[:200], flush=True)
