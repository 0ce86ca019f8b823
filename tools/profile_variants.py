#!/usr/bin/env python3
"""Launches chosen kernel variants once each (for ncu).  usage:
   profile_variants.py LOG2_COUNT kernel:unroll:preset[:threads] ..."""
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1902_05320_b200 import Engine  # noqa: E402

count = 1 << int(sys.argv[1])
e = Engine()
dev = e.generate_workload(count * 64, 64, seed=1)
out = torch.empty((count, 32), dtype=torch.uint8, device="cuda")
for spec in sys.argv[2:]:
    f = [int(x) for x in spec.split(":")]
    eng = Engine(kernel=f[0], unroll=f[1], fma_preset=f[2], block_threads=f[3] if len(f) > 3 else 0)
    for _ in range(2):
        eng.hash_fixed("sha3_256", dev, 64, count, out=out)
    torch.cuda.synchronize()
    print("ran", spec)
