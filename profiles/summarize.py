"""Summarise ncu captures into the committed profile notes.

    python profiles/summarize.py gpurun_out/prof_chain.ncu-rep [--launches gpurun_out/launches.csv]

Prints (markdown) the metrics DESIGN.md / bench.py cite: duration, tensor /
XU / FMA / ALU pipe activity, issue activity, DRAM bytes (the roofline
`traffic`), warp-stall breakdown, the dynamic opcode mix, and — for a
launch list — per-kernel share of device time.
"""
from __future__ import annotations

import csv
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration (us)"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (GHz)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU/conv) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
]


def ncu_csv(rep: str, *args: str) -> list[list[str]]:
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def summarize(rep: str) -> None:
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")]
    print(f"### {name}\n")
    print("| metric | value |\n|---|---|")
    for k, label in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"| {label} (`{k}`) | {vals[i]} {units[i]} |")
    stalls = [(h, vals[i]) for i, h in enumerate(hdr)
              if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio")]
    if stalls:
        print("\nwarp stall (cycles per issued instruction):\n")
        for h, v in sorted(stalls, key=lambda x: -float(x[1] or 0))[:8]:
            print(f"- {h.split('stalled_')[1].replace('.ratio', '')}: {v}")
    op = ncu_csv(rep, "--page", "raw", "--metrics", "sass__inst_executed_per_opcode",
                 "--print-metric-instances", "details")
    if len(op) >= 3:
        cell = op[-1][-1]
        if "(" in cell:
            mix = cell[cell.index("(") + 1: cell.rindex(")")].split(";")
            print("\ndynamic opcode mix (top 14):", ", ".join(m.strip() for m in mix[:14]))
    print()


def launches(path: str) -> None:
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    iK, iV, iM = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[iM] != "gpu__time_duration.sum":
            continue
        k = r[iK].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += float(r[iV].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | avg (us) | share of device time |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {t / n / 1e3:.2f} | {100 * t / tot:.1f}% |")
    print()


if __name__ == "__main__":
    args = sys.argv[1:]
    if "--launches" in args:
        i = args.index("--launches")
        launches(args[i + 1])
        del args[i: i + 2]
    for rep in args:
        summarize(rep)
