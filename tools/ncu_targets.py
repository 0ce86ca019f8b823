#!/usr/bin/env python3
"""Small launches for `ncu --set full` captures of the round-2 kernels (run under ncu with
-k regex:<kernel>): `fewblock` = three static multi-block shapes at 2^22 messages; `warp` = 256 x 256 KiB through the warp-per-state kernel; `short` = 2^22
ragged single-block messages at odd addresses (word-count order + jump-table absorb) and at
8-byte aligned addresses (input order, predicated absorb)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from paper_1902_05320_b200 import Engine  # noqa: E402

what = sys.argv[1]
eng = Engine(device=0)
if what == "fewblock":  # static multi-block shapes: SHAKE256 64 B -> 4096 bits, SHA3-384 256 B, SHA3-512 1 KiB
    count = 1 << 22
    shapes = (("shake256", 64, 4096), ("sha3_384", 256, 0), ("sha3_512", 1024, 0))
    if len(sys.argv) > 2 and sys.argv[2] == "xof":
        shapes = (("shake128", 64, 4096), ("shake256", 64, 4096), ("shake128", 64, 2048), ("shake256", 64, 2048))
    for alg, msg, bits in shapes:
        data = eng.generate_workload(count * msg, msg, seed=1)
        for _ in range(2):
            eng.hash_fixed(alg, data, msg, count, bits)
elif what == "warp":
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
