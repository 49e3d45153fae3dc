"""bench.py's contract on CPU: the configurations are BASELINE.json's, the FLOP / byte model is the
one SURVEY.md §8(d) states, and the reference arm (`--impl reference`, the reference's own CPU path)
prints one well-formed JSON line (no GPU needed)."""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_configs_are_baselines():
    cfgs = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    assert len(cfgs) == len(bench.CONFIGS) == 5
    for text, name in zip(cfgs, ("c1", "c2", "c3", "c4", "c5")):
        Bo, N, L, H, D, dt, _ = bench.CONFIGS[name]
        nums = {k: int(v) for k, v in re.findall(r"\b(N_seq|N_res|H|D)=(\d+)", text)}
        assert nums["H"] == H and nums["D"] == D and nums["N_res"] == L
        if "N_seq" in nums:
            assert nums["N_seq"] == N  # MSA rows
        else:
            assert N == L  # triangle attention: the start nodes are the rows
        assert ("fp32" in text) == (dt == "f32")


def test_flop_and_byte_model():
    B, L, H, D = 512, 384, 8, 32
    assert bench.flops(B, L, H, D) == 14 * B * H * L * L * D  # forward 4, backward 10 (§8(d))
    a_fwd, a_bwd = bench.algorithmic(B, L, H, D, 2)
    row = B * L * H * D * 2
    assert a_fwd["flop"] == 4 * B * H * L * L * D and a_bwd["flop"] == 10 * B * H * L * L * D
    assert a_bwd["bytes"] >= 8 * row  # Q, K, V, O, dO read; dQ, dK, dV written
    assert a_fwd["bytes"] >= 4 * row  # Q, K, V read; O written


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "TFLOP/s"
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
