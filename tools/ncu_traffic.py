#!/usr/bin/env python3
"""profiles/roofline_traffic.json from an `ncu --set full` capture of bench.py's own launch:
DRAM bytes read + written by ONE launch of the headline kernel, and the ALU-pipe instruction
count per message that the same capture measured.

usage: ncu_traffic.py REPORT.ncu-rep [MESSAGES_PER_LAUNCH] [OUT.json]

The capture (under gpurun; bench values are never taken from a run under ncu):
    ncu --set full --clock-control none --import-source on -k regex:hash_oneblock -s 3 -c 1 \
        -o gpurun_out/r2_oneblock_2p28 python bench.py --steps 1 --warmup 3 --no-e2e \
        --no-cpu-baseline --no-configs --no-dropin --no-probe
"""
import csv
import io
import json
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent


def to_bytes(value, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(value.replace(",", "")) * scale[unit]


def main():
    rep = sys.argv[1]
    messages = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
    out = pathlib.Path(sys.argv[3]) if len(sys.argv) > 3 else ROOT / "profiles" / "roofline_traffic.json"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    r = data[-1]
    read = to_bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
    write = to_bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
    grid = int(r[idx["launch__grid_size"]].replace(",", ""))
    block = int(r[idx["launch__block_size"]].replace(",", ""))
    rec = {
        "kernel": r[idx["Kernel Name"]],
        "source": f"profiles/{pathlib.Path(rep).stem}.md (ncu --set full, one launch of {messages} messages: "
                  "bench.py's own launch size)",
        "grid_x_block": [grid, block],
        "dram_bytes_read_per_launch": read,
        "dram_bytes_write_per_launch": write,
        "messages_per_launch": messages,
        "dram_bytes_per_message": (read + write) / messages,
        "algorithmic_bytes_per_message": 96,
        "duration_under_ncu": f"{r[idx['gpu__time_duration.sum']]} {units[idx['gpu__time_duration.sum']]}",
    }
    key = "sm__inst_executed_pipe_alu.sum"
    if key in idx:
        warp_instr = float(r[idx[key]].replace(",", ""))
        rec["alu_pipe_thread_instr_per_message"] = warp_instr * 32 / messages
    assert grid * block >= messages > (grid - 1) * block, "MESSAGES_PER_LAUNCH does not match the captured grid"
    out.write_text(json.dumps(rec, indent=1) + "\n")
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
