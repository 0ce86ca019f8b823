#!/usr/bin/env python3
"""One device-entry call per layout on 2^24 ragged single-block messages (SHA3-256, lengths
0..135), for an ncu launch list (--metrics gpu__time_duration.sum): which passes the call is
made of and what each costs.  argv[1]: start alignment (1 or 8)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from paper_1902_05320_b200 import Engine  # noqa: E402

pack = int(sys.argv[1]) if len(sys.argv) > 1 else 8
eng = Engine(device=0)
count = 1 << 24
g = torch.Generator(device="cuda").manual_seed(3)
lengths = torch.randint(0, 136, (count,), generator=g, device="cuda", dtype=torch.int64)
padded = (lengths + pack - 1) // pack * pack
offsets = torch.cumsum(padded, 0) - padded
data = torch.randint(0, 256, (int(padded.sum().item()) + 16,), dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
for _ in range(3):
    eng.hash_batch("sha3_256", data, offsets, lengths)
torch.cuda.synchronize()
