"""Summarise an ncu report (read here, no GPU) into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof_v.ncu-rep profiles/r1_c2_full.md \
        [--traffic-key c2] [--launches gpurun_out/launches.csv]

Writes a markdown table of the metrics that matter for these HBM/ALU-bound
kernels and merges per-launch DRAM traffic into profiles/traffic.json
({workload: {kernel_role: bytes}}) which bench.py reports as roofline.traffic.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]

ROLE = [("norm_kernel", "norm"), ("quantize_kernel", "quantize"), ("reduce_kernel", "reduce_decode"),
        ("baseline_tree_kernel", "fp32_baseline")]


def role(name: str) -> str:
    for k, v in ROLE:
        if k in name:
            return v
    return name.split("(")[0][-40:]


def to_bytes(val: str, unit: str) -> float:
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(val.replace(",", "")) * mult


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--traffic-key")
    ap.add_argument("--title", default="")
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary{(' — ' + args.title) if args.title else ''}", "",
             f"Source: `{args.rep}` (ncu --set full --clock-control none --import-source on; "
             "cold-cache serialised replays — compare shares, not absolutes).", ""]
    kernels = []
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        kernels.append((role(name), name, r))
    lines.append("| metric | " + " | ".join(k[0] for k in kernels) + " |")
    lines.append("|---|" + "---|" * len(kernels))
    for m, label in METRICS:
        if m not in col:
            continue
        vals = []
        for _, _, r in kernels:
            v = r[col[m]]
            u = units[col[m]]
            vals.append(f"{v} {u}".strip())
        lines.append(f"| {label} (`{m}`) | " + " | ".join(vals) + " |")
    lines.append("")
    for rl, name, _ in kernels:
        lines.append(f"- `{rl}`: `{name[:160]}`")
    Path(args.out).write_text("\n".join(lines) + "\n")
    if args.traffic_key:
        tp = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
        t = json.loads(tp.read_text()) if tp.exists() else {}
        ent = t.setdefault(args.traffic_key, {})
        for rl, _, r in kernels:
            b = to_bytes(r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]]) + \
                to_bytes(r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]])
            ent[rl] = b
        # the compute side of the same capture: issue-slot utilisation per kernel
        iss = t.setdefault("issue_active_pct", {}).setdefault(args.traffic_key, {})
        for rl, _, r in kernels:
            m = "smsp__issue_active.avg.pct_of_peak_sustained_active"
            if m in col:
                iss[rl] = float(r[col[m]])
        tp.write_text(json.dumps(t, indent=1, sort_keys=True) + "\n")
    print(Path(args.out).read_text())


if __name__ == "__main__":
    main()
