#!/usr/bin/env python3
"""Condenses ncu launch lists (`ncu --metrics gpu__time_duration.sum --clock-control none --csv`)
into one markdown file: per kernel, launches, total and average duration, share of the run.
usage: launch_summary.py OUT.md TITLE=list.csv [TITLE=list.csv ...]"""
import collections
import csv
import sys


def table(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    agg = collections.OrderedDict()
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "").replace("b200sha3::", "").replace("<unnamed>::", "").strip()
        if len(name) > 90:
            name = "..." + name[-87:]
        slot = agg.setdefault(name, [0, 0.0])
        slot[0] += 1
        slot[1] += float(r[-1])
    total = sum(v[1] for v in agg.values())
    out = [f"{len(rows)} launches, {total / 1e6:.3f} ms of kernel time in all.", "",
           "| kernel | launches | total ms | average ms | share |", "|---|---|---|---|---|"]
    for name, (n, ns) in agg.items():
        out.append(f"| `{name}` | {n} | {ns / 1e6:.3f} | {ns / n / 1e6:.4f} | {100 * ns / total:.1f} % |")
    return out


def main():
    lines = ["# ncu launch lists, round 2", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none --csv` over `bench.py` (per-launch",
             "times under ncu are serialised and cold-cache; the SHARES are what they are for).", ""]
    for arg in sys.argv[2:]:
        title, path = arg.split("=", 1)
        lines += [f"## {title}", ""] + table(path) + [""]
    open(sys.argv[1], "w").write("\n".join(lines))
    print("wrote", sys.argv[1])


if __name__ == "__main__":
    main()
