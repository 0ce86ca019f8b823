#!/usr/bin/env python3
"""Register-bank census of the round loops in libb200sha3.so (no GPU needed).

A LOP3 / SHF reads up to three registers; when all three sit in the same register bank (bank =
register number mod 2 on this architecture, as far as the timings below tell) the operand fetch
takes an extra cycle unless the operand-reuse cache helps.  Where ptxas keeps the 50 state
registers decides how many instructions of a round loop are in that position: 1-11 of 540 in a
good allocation, 65-87 in a bad one -- measured ~1.5-2 % slower (hash_fewblock_kernel<21, 8, 128>:
87 -> 0.989 of the ALU roofline, 1 -> 1.006; <17, 8, 128>: 66-70 -> 0.992-0.995, 11 -> 1.003).  The
allocation reacts to details far from the loop (the form of the output stores), so the store form
of kernel_fewblock.cu is picked per shape with this census.

    python tools/sass_bank_census.py [object or library ...]   (default: the built library)

Per kernel: ALU instructions (LOP3 + SHF) inside the innermost backward-branch loop, how many of
them read three registers of one parity, how many carry a .reuse flag.
"""
import pathlib
import re
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
INSTR = re.compile(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);")
TARGET = re.compile(r"0x([0-9a-f]+)")


def census(path):
    out = subprocess.run(["cuobjdump", "-sass", str(path)], capture_output=True, text=True, check=True).stdout
    funcs, name = {}, None
    for line in out.splitlines():
        if "Function :" in line:
            name = line.split("Function :")[1].strip()
            funcs[name] = []
            continue
        m = INSTR.match(line)
        if m and name:
            funcs[name].append((int(m.group(1), 16), m.group(2).strip()))
    names = list(funcs)
    pretty = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    rows = []
    for name, shown in zip(names, pretty):
        ins = funcs[name]
        loops = []
        for addr, text in ins:
            if text.split()[0].startswith("BRA") or (text.startswith("@") and "BRA" in text.split()[1]):
                m = TARGET.search(text)
                if m and int(m.group(1), 16) < addr:
                    loops.append((addr - int(m.group(1), 16), int(m.group(1), 16), addr))
        if not loops:
            continue
        _, lo, hi = max(loops)          # the largest loop: the round loop
        alu = same = reuse = 0
        for addr, text in ins:
            if not (lo <= addr <= hi):
                continue
            body = text.split(None, 1)[1] if text.startswith("@") else text
            if not (body.startswith("LOP3") or body.startswith("SHF")):
                continue
            alu += 1
            srcs = [o.strip() for o in body.split(None, 1)[1].split(",")[1:]]
            regs = [int(re.match(r"R(\d+)", x).group(1)) for x in srcs if re.match(r"R\d+", x)]
            reuse += any(".reuse" in x for x in srcs)
            if len(regs) >= 3 and len({r % 2 for r in regs}) == 1:
                same += 1
        short = re.sub(r"\(.*", "", shown.replace("void ", "").replace("b200sha3::", "").replace("(anonymous namespace)::", ""))
        rows.append((short, alu, same, reuse))
    return rows


def main():
    paths = sys.argv[1:] or [ROOT / "paper_1902_05320_b200" / "libb200sha3.so"]
    print("| kernel | ALU instructions in the round loop | three sources in one bank | with .reuse |")
    print("|---|---|---|---|")
    for path in paths:
        for short, alu, same, reuse in census(path):
            if alu >= 100:
                print(f"| `{short}` | {alu} | {same} | {reuse} |")


if __name__ == "__main__":
    main()
