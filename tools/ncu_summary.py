#!/usr/bin/env python3
"""Condenses an .ncu-rep (ncu --set full) into a small markdown table + stall table.
usage: ncu_summary.py REPORT.ncu-rep OUT.md"""
import csv
import io
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slot busy %"),
    ("sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active", "ALU pipe % (LOP3+SHF)"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA-heavy pipe % (IMAD)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__cycles_elapsed.max.per_second", "SM clock"),
]
STALLS = ["math_pipe_throttle", "not_selected", "wait", "no_instruction", "dispatch_stall",
          "long_scoreboard", "short_scoreboard", "lg_throttle"]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary of `{rep.split('/')[-1]}`", "",
             "`ncu --set full --clock-control none --import-source on`; one column per captured launch.", ""]
    names = []
    for r in data:
        n = r[idx["Kernel Name"]]
        m = re.search(r"(\w+_kernel)<([^>]*)>", n)
        names.append(f"{m.group(1)}<{m.group(2)}>".replace("(int)", "").replace("(unsigned int)", "")
                     if m else n[:50])
    lines.append("| metric | " + " | ".join(names) + " |")
    lines.append("|---|" + "---|" * len(names))
    for key, label in METRICS:
        if key not in idx:
            continue
        vals = [f"{r[idx[key]]} {units[idx[key]]}".strip() for r in data]
        lines.append(f"| {label} (`{key}`) | " + " | ".join(vals) + " |")
    lines += ["", "Warp stall reasons (`smsp__average_warps_issue_stalled_*_per_issue_active.ratio`):", "",
              "| stall | " + " | ".join(names) + " |", "|---|" + "---|" * len(names)]
    for s in STALLS:
        key = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if key in idx:
            lines.append(f"| {s} | " + " | ".join(f"{float(r[idx[key]]):.2f}" for r in data) + " |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
