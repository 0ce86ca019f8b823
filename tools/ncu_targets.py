#!/usr/bin/env python3
"""Small launches for `ncu --set full` captures of the round-2 kernels (run under ncu with
-k regex:<kernel>): `warp` = 256 x 256 KiB through the warp-per-state kernel; `short` = 2^22
ragged single-block messages at odd addresses (word-count order + jump-table absorb) and at
8-byte aligned addresses (input order, predicated absorb)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from paper_1902_05320_b200 import Engine  # noqa: E402

what = sys.argv[1]
eng = Engine(device=0)
if what == "warp":
    count, msg = 256, 256 << 10
    data = eng.generate_workload(count * msg, msg, seed=1)
    for _ in range(3):
        eng.hash_fixed("sha3_256", data, msg, count)
else:
    count = 1 << 22
    g = torch.Generator(device="cuda").manual_seed(3)
    lengths = torch.randint(0, 136, (count,), generator=g, device="cuda", dtype=torch.int64)
    for pack in (1, 8):
        padded = (lengths + pack - 1) // pack * pack
        offsets = torch.cumsum(padded, 0) - padded
        data = torch.randint(0, 256, (int(padded.sum().item()) + 16,), dtype=torch.uint8, device="cuda")
        for _ in range(2):
            eng.hash_batch("sha3_256", data, offsets, lengths)
torch.cuda.synchronize()
