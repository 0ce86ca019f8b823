#!/usr/bin/env python3
"""Equal-length batches whose length is NOT a whole number of lanes (the paper's 10-byte
messages) on the device entry: device time vs the ALU peak.  SHA3-256, 2^24 messages."""
import json
import pathlib
import sys

import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1902_05320_b200 import Engine  # noqa: E402

engine = Engine(device=0)
peak, _ = engine.probe_pipe(2)
count = 1 << 24
out = []
for msg_len in (10, 20, 33, 64, 100, 135):
    data = torch.randint(0, 256, (count * msg_len + 16,), dtype=torch.uint8, device="cuda")
    best = None
    for _ in range(5):
        engine.hash_fixed("sha3_256", data, msg_len, count, timed=True)
        best = engine.last_device_ms if best is None else min(best, engine.last_device_ms)
    rec = {"message_bytes": msg_len, "messages": count, "device_ms": best, "ghash_per_s": count / best / 1e6,
           "int_roofline_frac": count / (best * 1e-3) * 4320 / peak}
    out.append(rec)
    print(json.dumps(rec), flush=True)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "fixed_odd_lengths.json").write_text(json.dumps(out, indent=1))
