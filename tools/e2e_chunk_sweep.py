#!/usr/bin/env python3
"""e2e (host-buffer entry) throughput vs pipeline chunk size.  Runs bench.py once per
B200SHA3_CHUNK_MIB value; writes gpurun_out/e2e_chunks.json."""
import json
import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
out = []
for mib in [int(x) for x in (sys.argv[1:] or ["16", "32", "64", "128", "256"])]:
    env = dict(os.environ, B200SHA3_CHUNK_MIB=str(mib))
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline", "--no-probe", "--e2e-steps", "4"],
                       capture_output=True, text=True, env=env)
    line = json.loads(r.stdout.strip().splitlines()[-1])
    rec = {"chunk_mib": mib, "e2e_ghash_per_s": line["e2e"]["value"] / 1e9, **line["e2e"]["pcie"]}
    rec.pop("note", None)
    out.append(rec)
    print(rec, flush=True)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "e2e_chunks.json").write_text(json.dumps(out, indent=1))
