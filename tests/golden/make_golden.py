#!/usr/bin/env python3
"""Converts the reference's on-disk KAT fixtures into tests/golden/*.kat.

Run in the build container, where the reference is mounted:

    python tests/golden/make_golden.py [/root/reference]

Source: <ref>/proj/tests/vectors/*.rsp (12 files, 892 vectors; NIST-style
`Len = <bits>` / `Msg = <hex>` / `MD = <hex>` records under an `[L = n]` or
`[Outputlen = n]` header -- format per proj/tools/sha3cli/vectors.hpp:42-45).
The GPU box has no /root/reference, so the vectors travel as these committed
fixtures.  Output format, one vector per line:

    <len_bits> <msg_hex or "-" when empty> <digest_hex>

with a first line `# algorithm=<0..5> output_bits=<n> source=<file> vectors=<k>`.
Algorithm ids follow the reference enum (proj/core/include/sha3/sha3.hpp:15-22).
Nothing is recomputed here: message and digest hex are carried over verbatim.
"""
import pathlib
import re
import sys

ALGORITHM_ID = {"SHA3_224": 0, "SHA3_256": 1, "SHA3_384": 2, "SHA3_512": 3,
                "SHAKE128": 4, "SHAKE256": 5}


def parse_rsp(path: pathlib.Path):
    out_bits = None
    records, cur = [], {}
    for raw in path.read_text().splitlines():
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        m = re.fullmatch(r"\[(L|Outputlen)\s*=\s*(\d+)\]", line)
        if m:
            out_bits = int(m.group(2))
            continue
        key, _, value = (s.strip() for s in line.partition("="))
        cur[key] = value
        if key == "MD":
            nbits = int(cur["Len"])
            msg = cur["Msg"] if nbits else ""
            assert len(msg) == nbits // 4, (path, nbits)
            records.append((nbits, msg.lower(), cur["MD"].lower()))
            cur = {}
    return out_bits, records


def main():
    ref = pathlib.Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference")
    src = ref / "proj" / "tests" / "vectors"
    here = pathlib.Path(__file__).parent
    total = 0
    for rsp in sorted(src.glob("*.rsp")):
        label = re.match(r"(SHA3_\d+|SHAKE\d+)", rsp.name).group(1)
        out_bits, records = parse_rsp(rsp)
        dst = here / (rsp.stem + ".kat")
        with open(dst, "w") as f:
            f.write(f"# algorithm={ALGORITHM_ID[label]} output_bits={out_bits} "
                    f"source=proj/tests/vectors/{rsp.name} vectors={len(records)}\n")
            for nbits, msg, md in records:
                f.write(f"{nbits} {msg or '-'} {md}\n")
        total += len(records)
        print(f"{dst.name}: {len(records)} vectors")
    print("total", total)


if __name__ == "__main__":
    main()
