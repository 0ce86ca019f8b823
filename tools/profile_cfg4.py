#!/usr/bin/env python3
"""One bucketed + one unbucketed launch of the generic kernel on a cfg4-shaped batch
(lengths 1..16 KiB) for ncu.  usage: profile_cfg4.py LOG2_COUNT"""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1902_05320_b200 import Engine  # noqa: E402
from paper_1902_05320_b200.engine import FLAG_NO_BUCKETING  # noqa: E402

count = 1 << int(sys.argv[1])
e = Engine()
lengths = e.generate_lengths(count, 1, 16384, seed_len=2)
padded = (lengths + 7) // 8 * 8
offsets = torch.cumsum(padded, 0) - padded
data = torch.empty(int(padded.sum().item()) + 16, dtype=torch.uint8, device="cuda")
e.fill_messages(data, offsets, lengths, seed=1)
out = torch.empty((count, 32), dtype=torch.uint8, device="cuda")
for eng in (e, Engine(flags=FLAG_NO_BUCKETING)):
    for _ in range(2):
        eng.hash_batch("sha3_256", data, offsets, lengths, out=out)
    torch.cuda.synchronize()
print("bytes", int(lengths.sum().item()), "perms", int((lengths // 136 + 1).sum().item()))
