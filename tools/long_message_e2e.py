#!/usr/bin/env python3
"""Few long equal-length messages through the HOST entry (pinned buffers, wall clock): the piece
pipeline of b200sha3_hash_fixed (strided copies + incremental warp kernel) against the same call
without the pipeline (one copy, one launch) and against the plain H2D copy of the batch.
usage: long_message_e2e.py [count=1024] [message_KiB=1024]"""
import json
import pathlib
import sys
import time

import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1902_05320_b200 import Engine  # noqa: E402
from paper_1902_05320_b200.engine import FLAG_NO_PIPELINE, FLAG_NO_WARP_KERNEL  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
msg = (int(sys.argv[2]) if len(sys.argv) > 2 else 1024) << 10
host = torch.randint(0, 256, (count * msg,), dtype=torch.uint8).pin_memory()
out = torch.zeros(count * 32, dtype=torch.uint8).pin_memory()
dev = torch.empty(count * msg, dtype=torch.uint8, device="cuda")
rec = {"messages": count, "message_bytes": msg}
for name, eng in (("pieces", Engine()), ("one_copy_one_launch", Engine(flags=FLAG_NO_PIPELINE)),
                  ("message_chunks_thread_kernel", Engine(flags=FLAG_NO_WARP_KERNEL))):
    times = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.hash_fixed_ptr("sha3_256", host.data_ptr(), msg, count, out.data_ptr())
        times.append(time.perf_counter() - t0)
    rec[name] = {"wall_ms": sorted(times)[len(times) // 2] * 1e3, "launches": eng.last_kernel_launches,
                 "digest0": bytes(out[:8].tolist()).hex()}
times = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    times.append(time.perf_counter() - t0)
rec["plain_h2d_ms"] = sorted(times)[2] * 1e3
print(json.dumps(rec, indent=1))
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / f"long_message_e2e_{count}x{msg >> 10}KiB.json").write_text(json.dumps(rec, indent=1))
