#!/usr/bin/env python3
"""Few, long messages: device time of one hash_batch_device launch vs the number of messages
(one message is one thread; the sponge is sequential per message).  SHA3-256.
usage: long_message_latency.py [message_KiB=1024] [block_threads ...]"""
import json
import pathlib
import sys

import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1902_05320_b200 import Engine  # noqa: E402

kib = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
blocks = [int(x) for x in sys.argv[2:]] or [0]
msg = kib << 10
out = []
for bt in blocks:
    engine = Engine(device=0, block_threads=bt)
    for count in (32, 128, 256, 512, 1024, 2048, 4096, 8192):
        if count * msg > (24 << 30):
            break
        data = torch.randint(0, 256, (count * msg,), dtype=torch.uint8, device="cuda")
        offsets = (torch.arange(count, dtype=torch.int64, device="cuda") * msg)
        lengths = torch.full((count,), msg, dtype=torch.int64, device="cuda")
        best = None
        for _ in range(3):
            engine.hash_batch("sha3_256", data, offsets, lengths, timed=True)
            ms = engine.last_device_ms
            best = ms if best is None else min(best, ms)
        perms = msg // 136 + 1
        rec = {"block_threads": bt, "messages": count, "message_KiB": kib, "device_ms": best,
               "us_per_permutation_per_thread": best * 1e3 / perms, "GB_per_s": count * msg / best / 1e6}
        out.append(rec)
        print(json.dumps(rec), flush=True)
        del data
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / f"long_message_latency_{kib}KiB.json").write_text(json.dumps(out, indent=1))
