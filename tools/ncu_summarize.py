"""Summarise ncu captures into the committed profiles/ directory.

  python tools/ncu_summarize.py launches <launches.csv> <out.md> [--config c4]
      per-kernel launch list of one bench command (gpu__time_duration.sum, cold-cache, serialised):
      each kernel's count, mean duration and share of the captured steps.
  python tools/ncu_summarize.py full <report.ncu-rep> <out.md> [--config c4] [--traffic profiles/ncu_traffic.json]
      key counters of every kernel in a `ncu --set full` capture (duration, DRAM bytes, tensor-pipe
      and issue utilisation, shared-memory wavefronts, top stall reasons); DRAM bytes per launch are
      merged into the traffic JSON read by bench.py (roofline.traffic).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "LSU shared wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "tensor-core shared wavefronts"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel)<([^>]*)>", name)
    return f"{m.group(1)}<{m.group(2)}>" if m else name.split("(")[0][:60]


def launches(path, out, config):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[short(r[ki])].append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    with open(out, "w") as f:
        f.write(f"# Launch list — bench.py --config {config} (ncu --metrics gpu__time_duration.sum --clock-control none)\n\n")
        f.write("Cold-cache, serialised per-launch times: compare SHARES with bench.py, not absolutes.\n\n")
        f.write("| kernel | launches | mean µs | total µs | share |\n|---|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / 1e3:.1f} | {sum(v) / total:.1%} |\n")
    print(open(out).read())


def full(rep, out, config, traffic_path):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    recs = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
    traffic, call = {}, {}
    if traffic_path and os.path.exists(traffic_path):
        traffic = json.load(open(traffic_path))
    with open(out, "w") as f:
        f.write(f"# ncu --set full — {config} ({os.path.basename(rep)})\n\n")
        for d in recs:
            name = short(d.get("Kernel Name", "?"))
            f.write(f"## `{name}`\n\n| counter | value |\n|---|---|\n")
            for k, label in KEYS:
                if k in d and d[k] not in ("", "n/a"):
                    f.write(f"| {label} (`{k}`) | {d[k]} |\n")
            stalls = {k.split("pcsamp_warps_issue_stalled_")[1]: float(d[k].replace(",", ""))
                      for k in d if "pcsamp_warps_issue_stalled_" in k and not k.endswith("not_issued")
                      and d[k] not in ("", "n/a")}
            tot = sum(stalls.values()) or 1
            top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
            f.write("\nTop warp-stall reasons (share of PC samples): "
                    + ", ".join(f"{k} {v / tot:.0%}" for k, v in top) + "\n\n")
            try:
                rd = float(d["dram__bytes_read.sum"].replace(",", ""))
                wr = float(d["dram__bytes_write.sum"].replace(",", ""))
                unit_r = h_units(rows, "dram__bytes_read.sum")
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit_r, 1)
                key = f"{config}_{'bwd' if 'bwd' in name else 'fwd'}_tcgen05"
                if "bwd_kernel" in name or "fwd_kernel" in name:
                    traffic[key] = (rd + wr) * mult
                if any(k in name for k in ("prep_kernel", "bwd_kernel", "dq_convert")):
                    call[name] = (rd + wr) * mult  # the backward call: preamble + main kernel + conversion
            except (KeyError, ValueError):
                pass
    if len(call) == 3:
        traffic[f"{config}_bwd_call_tcgen05"] = sum(call.values())
    if traffic_path:
        json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
    print(open(out).read())


def h_units(rows, key):
    h, units = rows[0], rows[1]
    return units[h.index(key)] if key in h else ""


if __name__ == "__main__":
    mode, src, out = sys.argv[1:4]
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "c4"
    tr = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    (launches if mode == "launches" else lambda a, b, c: full(a, b, c, tr))(src, out, cfg)
