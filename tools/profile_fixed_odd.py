#!/usr/bin/env python3
"""Two launches of the equal-length short kernel on 2^22 messages of LEN bytes, for ncu.
usage: profile_fixed_odd.py [LEN=10]"""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1902_05320_b200 import Engine  # noqa: E402

msg_len = int(sys.argv[1]) if len(sys.argv) > 1 else 10
count = 1 << 22
data = torch.randint(0, 256, (count * msg_len + 16,), dtype=torch.uint8, device="cuda")
e = Engine()
for _ in range(2):
    e.hash_fixed("sha3_256", data, msg_len, count)
torch.cuda.synchronize()
