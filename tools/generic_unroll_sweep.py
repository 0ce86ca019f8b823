#!/usr/bin/env python3
"""Loop shape of the generic kernel's permutation (rounds per body) on SHA3-256 1 KiB and
64 B messages.  Writes gpurun_out/generic_unroll.json."""
import json
import pathlib
import statistics
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1902_05320_b200 import Engine, permutations  # noqa: E402
from paper_1902_05320_b200.engine import KERNEL_GENERIC  # noqa: E402

res = []
peak, _ = Engine().probe_pipe(2)
for msg_len, log2 in ((1024, 24), (64, 24)):
    count = 1 << log2
    data = Engine().generate_workload(count * msg_len, msg_len, seed=1)
    ref = None
    for unroll in (0, 2, 4, 6):
        for threads in (128, 256):
            e = Engine(kernel=KERNEL_GENERIC, unroll=unroll, block_threads=threads)
            out = e.hash_fixed("sha3_256", data, msg_len, count)
            ref = out if ref is None else ref
            assert torch.equal(out, ref)
            ms = []
            for _ in range(5):
                e.hash_fixed("sha3_256", data, msg_len, count, out=out, timed=True)
                ms.append(e.last_device_ms)
            t = statistics.median(ms)
            perms = count * permutations("sha3_256", msg_len)
            res.append({"msg_len": msg_len, "rounds_per_body": unroll or 3, "threads": threads, "ms": t,
                        "int_roofline_frac": perms / t * 1e3 * 4320 / peak})
            print(res[-1], flush=True)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / "generic_unroll.json").write_text(json.dumps(res, indent=1))
