#!/usr/bin/env python3
"""Per-opcode warp-stall samples from the source page of an .ncu-rep (needs -lineinfo and
--import-source on).  usage: ncu_stalls_by_opcode.py REPORT.ncu-rep OUT.md [max_kernels]"""
import collections
import csv
import io
import re
import subprocess
import sys

STALLS = ["stall_math", "stall_not_selected", "stall_wait", "stall_selected", "stall_no_inst",
          "stall_dispatch", "stall_long_sb", "stall_short_sb", "stall_lg", "stall_branch_resolving"]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    limit = int(sys.argv[3]) if len(sys.argv) > 3 else 99
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    kernels, cur = [], None
    for r in csv.reader(io.StringIO(raw)):
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            kernels.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r:
            cur["rows"].append(r)
    lines = [f"# warp-stall samples by opcode, `{rep.split('/')[-1]}`", "",
             "Source page of `ncu --set full --import-source on` (sampled warp states, all samples).", ""]
    seen = set()
    for k in kernels:
        m = re.search(r"(\w+_kernel)<([^>]*)>", k["name"])
        name = f"{m.group(1)}<{m.group(2)}>".replace("(int)", "").replace("(unsigned int)", "") if m else k["name"][:60]
        if name in seen or len(seen) >= limit:
            continue
        seen.add(name)
        h = {n: i for i, n in enumerate(k["hdr"])}
        agg = collections.defaultdict(collections.Counter)
        for r in k["rows"]:
            toks = r[h["Source"]].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            key = op.split(".")[0] + (".HI" if ".HI" in op else "") + (".WIDE" if "WIDE" in op else "")
            agg[key]["instructions"] += 1
            for s in STALLS:
                v = r[h[s]] if s in h else ""
                agg[key][s] += int(v) if v else 0
        lines += [f"## `{name}`", "", "| opcode | static count | " + " | ".join(STALLS) + " |",
                  "|---|---|" + "---|" * len(STALLS)]
        for op, c in sorted(agg.items(), key=lambda kv: -sum(v for n, v in kv[1].items() if n != "instructions"))[:8]:
            lines.append(f"| {op} | {c['instructions']} | " + " | ".join(str(c[s]) for s in STALLS) + " |")
        lines.append("")
    open(out, "w").write("\n".join(lines))
    print("wrote", out)


if __name__ == "__main__":
    main()
