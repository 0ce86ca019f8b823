#!/usr/bin/env python3
"""Randomized differential run: the CUDA path (every entry point and kernel selection)
against the CPU oracle, for a wall-clock budget.  Test infrastructure (it imports the oracle, which
only code under tests/ may do); not collected by pytest.  usage: python tests/fuzz_parity.py SECONDS [SEED]
Writes gpurun_out/fuzz_parity.json; exits 1 on the first mismatch (after dumping the case)."""
import json
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.binding import Oracle  # noqa: E402
from paper_1902_05320_b200 import BatchHasher, Engine  # noqa: E402
from paper_1902_05320_b200.engine import (FLAG_NO_BUCKETING, FLAG_NO_PIPELINE, FLAG_NO_WARP_KERNEL,  # noqa: E402
                                          KERNEL_AUTO, KERNEL_GENERIC, KERNEL_PAIR, KERNEL_STAGED, KERNEL_WARP)


def random_lengths(rng, count, rate):
    kind = rng.integers(0, 5)
    if kind == 0:
        return rng.integers(0, 64, count)
    if kind == 1:
        return rng.integers(0, 6 * rate, count)
    if kind == 2:  # hug the block boundaries
        return np.maximum(0, rng.integers(0, 8, count) * rate + rng.integers(-3, 4, count))
    if kind == 3:
        return np.full(count, rng.integers(0, 5 * rate))
    return np.where(rng.random(count) < 0.05, rng.integers(0, 40000, count), rng.integers(0, 300, count))


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    oracle = Oracle()
    stats = {"seed": seed, "cases": 0, "messages": 0, "bytes": 0, "by_entry": {}}
    t_end = time.time() + budget
    while time.time() < t_end:
        alg = int(rng.integers(0, 6))
        rate = oracle.rate_bytes(alg)
        bits = 0 if alg < 4 else int(rng.choice([1, 8, 12, 256, 328, 8 * rate, 8 * rate + 8, 3 * 8 * rate + 5, 4099]))
        count = int(rng.choice([1, 2, 31, 32, 33, 500, 4000]))
        lengths = random_lengths(rng, count, rate).astype(np.uint64)
        align = int(rng.choice([1, 1, 4, 8, 16]))
        lead = int(rng.integers(0, 16)) if align == 1 else 0
        offsets = np.zeros(count, dtype=np.uint64)
        pos = lead
        for i in range(count):
            pos += (-(pos - lead)) % align
            offsets[i] = pos
            pos += int(lengths[i])
        data = rng.integers(0, 256, pos + 16, dtype=np.uint8)
        expect = oracle.hash_batch(alg, data, offsets, lengths, xof_bits=bits, workers=8)
        entry = str(rng.choice(["device", "device_nobucket", "device_staged", "device_warp", "device_pair", "host", "host_nopipe",
                                "fixed_device", "fixed_host", "incremental"]))
        # small batches take the warp-per-state kernel by default: half of the cases switch it off
        # so that the one-message-per-thread kernels see small batches too
        no_warp = FLAG_NO_WARP_KERNEL if rng.random() < 0.5 else 0
        if entry.startswith("fixed"):
            n = int(lengths[0])
            if rng.random() < 0.35:  # the static multi-block shapes (kernel_fewblock.cu) and their neighbours
                n = int(rng.choice([128, 256, 512, 1024])) if alg < 4 else 64
                bits = 0 if alg < 4 else int(rng.choice([2048, 4096, 2045]))
                n += int(rng.choice([0, 0, 0, 8, -8]))
                if rng.random() < 0.3:  # any whole number of lanes (hash_manyblock_kernel when >= rate)
                    n = 8 * int(rng.integers(1, 6 * rate // 8 + 2))
                entry += "_shape"
            fixed = rng.integers(0, 256, max(count * n, 1) + 16, dtype=np.uint8)
            expect = oracle.hash_batch(alg, fixed, fixed_len=n, count=count, xof_bits=bits, workers=8)
            kernel = int(rng.choice([KERNEL_AUTO, KERNEL_AUTO, KERNEL_GENERIC, KERNEL_STAGED, KERNEL_WARP, KERNEL_PAIR]))
            eng = Engine(kernel=kernel, flags=no_warp)
            if entry.startswith("fixed_device"):
                got = eng.hash_fixed(alg, torch.from_numpy(fixed).cuda(), n, count, bits).cpu().numpy()
            else:
                got = eng.hash_fixed(alg, fixed, n, count, bits)
        elif entry == "incremental":
            h = BatchHasher(alg, count)
            d = torch.from_numpy(data).cuda()
            cut = (lengths * np.uint64(rng.integers(0, 101)) // np.uint64(100)).astype(np.int64)
            o = torch.from_numpy(offsets.astype(np.int64)).cuda()
            h.update(d, o, torch.from_numpy(cut).cuda())
            h.update(d, o + torch.from_numpy(cut).cuda(), torch.from_numpy(lengths.astype(np.int64) - cut).cuda())
            got = (h.digest() if alg < 4 else h.finish(bits)).cpu().numpy()
            h.close()
        elif entry.startswith("device"):
            flags = (FLAG_NO_BUCKETING if entry == "device_nobucket" else 0) | no_warp
            kernel = {"device_staged": KERNEL_STAGED, "device_warp": KERNEL_WARP, "device_pair": KERNEL_PAIR}.get(entry, KERNEL_AUTO)
            eng = Engine(flags=flags, kernel=kernel)
            got = eng.hash_batch(alg, torch.from_numpy(data).cuda(), torch.from_numpy(offsets.astype(np.int64)).cuda(),
                                 torch.from_numpy(lengths.astype(np.int64)).cuda(), bits).cpu().numpy()
        else:
            eng = Engine(flags=(FLAG_NO_PIPELINE if entry == "host_nopipe" else 0) | no_warp)
            got = eng.hash_batch(alg, data, offsets, lengths, bits)
        if not (got == expect).all():
            bad = int(np.argwhere((got != expect).any(axis=1))[0][0])
            print("MISMATCH", dict(entry=entry, alg=alg, bits=bits, count=count, align=align, lead=lead,
                                   message=bad, length=int(lengths[bad]), offset=int(offsets[bad])))
            sys.exit(1)
        stats["cases"] += 1
        stats["messages"] += count
        stats["bytes"] += int(lengths.sum())
        stats["by_entry"][entry] = stats["by_entry"].get(entry, 0) + 1
    stats["seconds"] = budget
    print(json.dumps(stats))
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "fuzz_parity.json").write_text(json.dumps(stats, indent=1))


if __name__ == "__main__":
    main()
