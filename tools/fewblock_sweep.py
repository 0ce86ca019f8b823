#!/usr/bin/env python3
"""Static multi-block shapes (kernel_fewblock.cu) next to the generic kernel, per block size:
device time (median of 5) and fraction of the measured ALU roofline on 2^24 messages."""
import json
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from paper_1902_05320_b200 import Engine, digest_bytes, permutations  # noqa: E402
from paper_1902_05320_b200.engine import KERNEL_FEWBLOCK, KERNEL_GENERIC  # noqa: E402

count = 1 << 24
probe = Engine(device=0)
peak, hz = probe.probe_pipe(2)
rows = []
shapes = [("shake128", 64, 2048), ("shake128", 64, 4096), ("shake256", 64, 2048), ("shake256", 64, 4096),
          ("sha3_224", 256, 0), ("sha3_384", 128, 0), ("sha3_384", 256, 0), ("sha3_512", 128, 0), ("sha3_512", 1024, 0),
          # run-time-length form (hash_manyblock_kernel): lengths without a static instantiation
          ("sha3_256", 136, 0), ("sha3_256", 200, 0), ("sha3_256", 1000, 0), ("sha3_224", 400, 0), ("sha3_384", 104, 0),
          ("sha3_512", 200, 0), ("shake128", 1024, 256), ("shake256", 200, 512)]
for alg, msg, bits in shapes:
    data = probe.generate_workload(count * msg, msg, seed=1)
    out = torch.empty((count, digest_bytes(alg, bits)), dtype=torch.uint8, device="cuda")
    row = {"algorithm": alg, "msg_len": msg, "xof_bits": bits}
    for name, kernel in (("fewblock", KERNEL_FEWBLOCK), ("generic", KERNEL_GENERIC)):
        for threads in (64, 128, 256):
            eng = Engine(device=0, kernel=kernel, block_threads=threads)
            times = []
            for i in range(7):
                eng.hash_fixed(alg, data, msg, count, bits, out=out, timed=True)
                if i >= 2:
                    times.append(eng.last_device_ms)
            ms = statistics.median(times)
            row[f"{name}_{threads}"] = {"ms": round(ms, 4),
                                        "frac": round(count * permutations(alg, msg, bits) / ms * 1e3 * 4320 / peak, 4)}
    rows.append(row)
    print(json.dumps(row), flush=True)
    del data, out
json.dump({"alu_peak_instr_per_s": peak, "sm_hz": hz, "rows": rows}, open("gpurun_out/fewblock_sweep.json", "w"), indent=1)
