#!/usr/bin/env python3
"""Two bucketed launches of the generic kernel on a SHORT ragged batch (lengths 0..max_len, 8-byte
aligned starts) for ncu.  usage: profile_short_ragged.py LOG2_COUNT [MAX_LEN=135]"""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1902_05320_b200 import Engine  # noqa: E402

count = 1 << int(sys.argv[1])
max_len = int(sys.argv[2]) if len(sys.argv) > 2 else 135
g = torch.Generator(device="cuda").manual_seed(3)
lengths = torch.randint(0, max_len + 1, (count,), generator=g, device="cuda", dtype=torch.int64)
padded = (lengths + 7) // 8 * 8
offsets = torch.cumsum(padded, 0) - padded
data = torch.randint(0, 256, (int(padded.sum().item()) + 16,), dtype=torch.uint8, device="cuda")
out = torch.empty((count, 32), dtype=torch.uint8, device="cuda")
e = Engine()
for _ in range(2):
    e.hash_batch("sha3_256", data, offsets, lengths, out=out)
torch.cuda.synchronize()
print("bytes", int(lengths.sum().item()), "perms", int((lengths // 136 + 1).sum().item()))
