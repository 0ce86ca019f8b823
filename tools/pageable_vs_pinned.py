#!/usr/bin/env python3
"""Host-buffer entry (b200sha3_hash_fixed / b200sha3_hash_batch) on pageable vs pinned host memory:
wall clock per call, SHA3-256.  Writes gpurun_out/pageable_vs_pinned.json."""
import json
import pathlib
import sys
import time

import numpy as np
import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1902_05320_b200 import Engine  # noqa: E402

engine = Engine(device=0)
RESULTS = []
for log2_count, msg_len in [(20, 64), (24, 64), (18, 4096)]:
    count = 1 << log2_count
    dev = engine.generate_workload(count * msg_len, msg_len, seed=1, count=count)
    pinned_in = torch.empty(count * msg_len, dtype=torch.uint8).pin_memory()
    pinned_out = torch.empty(count * 32, dtype=torch.uint8).pin_memory()
    pinned_in.copy_(dev)
    pageable_in = pinned_in.numpy().copy()
    pageable_out = np.empty(count * 32, dtype=np.uint8)
    rec = {"count": count, "message_bytes": msg_len}
    for name, src, dst in (("pinned", pinned_in.data_ptr(), pinned_out.data_ptr()),
                           ("pageable", pageable_in.ctypes.data, pageable_out.ctypes.data)):
        engine.hash_fixed_ptr("sha3_256", src, msg_len, count, dst)
        times = []
        for _ in range(5):
            t0 = time.perf_counter()
            engine.hash_fixed_ptr("sha3_256", src, msg_len, count, dst)
            times.append(time.perf_counter() - t0)
        t = sorted(times)[2]
        rec[name] = {"wall_ms": t * 1e3, "hashes_per_s": count / t, "h2d_gb_per_s": count * msg_len / t / 1e9}
    rec["digests_equal"] = bool((pinned_out.numpy() == pageable_out).all())
    RESULTS.append(rec)
    print(json.dumps(rec), flush=True)
# the variable-length entry: 2^24 short ragged messages (0..128 B), packed at 8-byte aligned offsets
count = 1 << 24
g = torch.Generator().manual_seed(5)
lengths = torch.randint(0, 129, (count,), generator=g, dtype=torch.int64)
padded = (lengths + 7) // 8 * 8
offsets = torch.cumsum(padded, 0) - padded
total = int(padded.sum().item()) + 16
pin = {"data": torch.randint(0, 256, (total,), dtype=torch.uint8).pin_memory(),
       "offsets": offsets.pin_memory(), "lengths": lengths.pin_memory(),
       "out": torch.empty(count * 32, dtype=torch.uint8).pin_memory()}
page = {k: v.numpy().copy() for k, v in pin.items()}
rec = {"count": count, "message_bytes": "ragged 0..128", "entry": "b200sha3_hash_batch"}
outs = {}
for name, bufs in (("pinned", {k: v.numpy() for k, v in pin.items()}), ("pageable", page)):
    out = bufs["out"].reshape(count, 32)
    engine.hash_batch("sha3_256", bufs["data"], bufs["offsets"].view(np.uint64), bufs["lengths"].view(np.uint64), out=out)
    times = []
    for _ in range(5):
        t0 = time.perf_counter()
        engine.hash_batch("sha3_256", bufs["data"], bufs["offsets"].view(np.uint64), bufs["lengths"].view(np.uint64),
                          out=out)
        times.append(time.perf_counter() - t0)
    t = sorted(times)[2]
    rec[name] = {"wall_ms": t * 1e3, "hashes_per_s": count / t}
    outs[name] = out
rec["digests_equal"] = bool((outs["pinned"] == outs["pageable"]).all())
print(json.dumps(rec), flush=True)
RAGGED = rec
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "pageable_vs_pinned.json").write_text(json.dumps(RESULTS + [RAGGED], indent=1))
