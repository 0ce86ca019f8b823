#!/usr/bin/env python3
"""Two launches of one fixed-length config (for ncu).  usage: profile_fixed.py ALG LEN LOG2 [BITS] [KERNEL]"""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1902_05320_b200 import Engine  # noqa: E402

alg, msg_len, log2 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
bits = int(sys.argv[4]) if len(sys.argv) > 4 else 0
kernel = int(sys.argv[5]) if len(sys.argv) > 5 else 0
count = 1 << log2
e = Engine(kernel=kernel)
dev = e.generate_workload(count * msg_len, msg_len, seed=1)
for _ in range(2):
    e.hash_fixed(alg, dev, msg_len, count, bits)
torch.cuda.synchronize()
print("ran", alg, msg_len, count)
