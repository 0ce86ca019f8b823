#!/usr/bin/env python3
"""Device entry on SHORT ragged batches (lengths uniform 0..max_len), SHA3-256: device time,
permutations/s against the measured ALU peak, with and without bucketing."""
import json
import pathlib
import sys

import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1902_05320_b200 import Engine  # noqa: E402
from paper_1902_05320_b200.engine import FLAG_NO_BUCKETING  # noqa: E402

probe = Engine(device=0)
peak, _ = probe.probe_pipe(2)
out = []
pack = int(sys.argv[1]) if len(sys.argv) > 1 else 8      # message starts are multiples of this
for log2_count, max_len in [(22, 300), (22, 1000), (20, 300), (24, 135), (22, 135), (22, 4096)]:
    count = 1 << log2_count
    g = torch.Generator(device="cuda").manual_seed(3)
    lengths = torch.randint(0, max_len + 1, (count,), generator=g, device="cuda", dtype=torch.int64)
    padded = (lengths + pack - 1) // pack * pack
    offsets = torch.cumsum(padded, 0) - padded
    data = torch.randint(0, 256, (int(padded.sum().item()) + 16,), dtype=torch.uint8, device="cuda")
    perms = int((lengths // 136 + 1).sum().item())
    rec = {"messages": count, "max_len": max_len, "start_alignment": pack, "permutations": perms}
    for name, flags in (("bucketed", 0), ("input_order", FLAG_NO_BUCKETING)):
        eng = Engine(device=0, flags=flags)
        best = None
        for _ in range(5):
            eng.hash_batch("sha3_256", data, offsets, lengths, timed=True)
            best = eng.last_device_ms if best is None else min(best, eng.last_device_ms)
        rec[name] = {"device_ms": best, "gperm_per_s": perms / best / 1e6,
                     "int_roofline_frac": perms / (best * 1e-3) * 4320 / peak}
    out.append(rec)
    print(f"align {pack}: 2^{log2_count} x 0..{max_len} B  bucketed {rec['bucketed']['int_roofline_frac']:.3f} "
          f"({rec['bucketed']['device_ms']:.3f} ms)  input order {rec['input_order']['int_roofline_frac']:.3f} "
          f"({rec['input_order']['device_ms']:.3f} ms)", flush=True)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / f"short_ragged_align{pack}.json").write_text(json.dumps(out, indent=1))
