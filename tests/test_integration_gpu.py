"""Drop-in check: the reference's own attn-bench harness (run.cpp, unmodified)
linked against integration/evomem_gpu_adapter.cpp instead of attention_tiled.cpp, so every
evomem::attn_forward_tiled / attn_backward_tiled call runs on the B200 kernels. The harness
compares against the reference's materialising oracle (attention.cpp) with its own tolerances
(run.cpp:116-126: F32 1e-5, BF16/F16 5e-2 max-abs) and exits 2 on a failed check.
The binary is prebuilt by `make -C integration` (needs /root/reference; travels in oracle/_ref/)."""
import csv
import io
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "oracle", "_ref", "evomem_gpu_harness")

pytestmark = pytest.mark.gpu


def _run(*args):
    if not os.path.exists(HARNESS):
        pytest.fail("integration harness not built (make -C integration, needs /root/reference)")
    return subprocess.run([HARNESS, *args], capture_output=True, text=True, timeout=600)


def test_reference_attn_bench_runs_on_gpu(cuda):
    r = _run("attn-bench", "--config", os.path.join(ROOT, "integration", "attn_bench_gpu.json"), "--seed", "0")
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert len(rows) == 9
    for row in rows:
        assert float(row["max_abs_diff"]) < 5e-2
        assert int(row["tiled_peak_bytes"]) < int(row["naive_peak_bytes"])  # no L x L logits
    f32 = [float(r_["max_abs_diff"]) for r_ in rows[:6]]
    assert max(f32) < 1e-5


def test_reference_error_contract_for_f64(cuda):
    # the default suite contains an F64 case: the adapter raises ValidationError -> exit code 1
    r = _run("attn-bench")
    assert r.returncode == 1
    assert "F64" in r.stderr
