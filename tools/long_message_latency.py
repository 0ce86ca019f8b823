#!/usr/bin/env python3
"""Few, long messages: device time of one b200sha3_hash_batch_device call against the number of
messages, for the one-message-per-thread path (FLAG_NO_WARP_KERNEL: bucketing + generic kernel)
and the warp-per-state kernel (KERNEL_WARP), SHA3-256.  The sponge is sequential per message,
so below a few thousand messages the time is (blocks per message) x (latency of one
permutation) and the two layouts differ in exactly that latency.  Finds the crossover that
capi.cu's warp_kernel_max_count() encodes.

usage: long_message_latency.py [message_KiB=1024] [max_count=8192]"""
import json
import pathlib
import sys

import torch

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1902_05320_b200 import Engine  # noqa: E402
from paper_1902_05320_b200.engine import FLAG_NO_WARP_KERNEL, KERNEL_GENERIC, KERNEL_PAIR, KERNEL_WARP  # noqa: E402

kib = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
max_count = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
name_of_sweep = sys.argv[3] if len(sys.argv) > 3 else "fine"   # "wide": counts double every step
msg = kib << 10
perms = msg // 136 + 1
peak, hz = Engine(device=0).probe_pipe(2)
engines = {"thread_per_message": Engine(device=0, kernel=KERNEL_GENERIC),
           "pair_per_message": Engine(device=0, kernel=KERNEL_PAIR),
           "warp_per_message": Engine(device=0, kernel=KERNEL_WARP)}
out = []
count = 32
while count <= max_count and count * msg <= (48 << 30):
    data = torch.randint(0, 256, (count * msg + 16,), dtype=torch.uint8, device="cuda")
    offsets = torch.arange(count, dtype=torch.int64, device="cuda") * msg
    lengths = torch.full((count,), msg, dtype=torch.int64, device="cuda")
    rec = {"messages": count, "message_KiB": kib, "permutations_per_message": perms}
    digests = {}
    for name, engine in engines.items():
        best = None
        if name == "warp_per_message" and count > 8192:
            continue                       # far beyond its range: minutes per launch
        for _ in range(4):
            digests[name] = engine.hash_batch("sha3_256", data, offsets, lengths, timed=True)
            best = engine.last_device_ms if best is None else min(best, engine.last_device_ms)
        rec[name] = {"device_ms": best, "us_per_permutation": best * 1e3 / perms,
                     "cycles_per_permutation": best * 1e-3 / perms * hz,
                     "GB_per_s_hashed": count * msg / best / 1e6,
                     "int_roofline_frac": count * perms / (best * 1e-3) * 4320 / peak}
    rec["digests_equal"] = all(bool(torch.equal(digests["thread_per_message"], d)) for d in digests.values())
    for other in ("pair_per_message", "warp_per_message"):
        if other in rec:
            rec[f"speedup_{other.split('_')[0]}_over_thread"] = rec["thread_per_message"]["device_ms"] / rec[other]["device_ms"]
    out.append(rec)
    print(count, {k: round(v["cycles_per_permutation"]) for k, v in rec.items() if isinstance(v, dict)},
          "equal" if rec["digests_equal"] else "DIGESTS DIFFER", flush=True)
    del data
    if name_of_sweep == "wide":
        count *= 2
    else:
        count = count * 2 if count < 1024 else count + (512 if count < 4096 else 2048)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / f"long_message_latency_{kib}KiB.json").write_text(
    json.dumps({"alu_peak_instr_per_s": peak, "sm_hz": hz, "rows": out}, indent=1))
