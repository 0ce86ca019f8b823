#!/usr/bin/env python3
"""Direct per-thread loads (generic kernel) vs TMA-staged blocks (staged kernel) on the
long-message configs.  Writes gpurun_out/staged_vs_direct.json."""
import json
import pathlib
import statistics
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1902_05320_b200 import Engine, permutations  # noqa: E402
from paper_1902_05320_b200.engine import KERNEL_GENERIC, KERNEL_STAGED  # noqa: E402


def med(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    return statistics.median(fn() for _ in range(reps))


def main():
    res = []
    peak, _ = Engine().probe_pipe(2)
    engines = {"direct (generic)": Engine(kernel=KERNEL_GENERIC), "TMA-staged": Engine(kernel=KERNEL_STAGED)}
    for alg, msg_len, log2 in (("sha3_256", 1024, 24), ("sha3_512", 1024, 24), ("shake128", 4096, 22)):
        count = 1 << log2
        data = engines["TMA-staged"].generate_workload(count * msg_len, msg_len, seed=1)
        bits = 256 if alg.startswith("shake") else 0
        outs = {}
        for name, e in engines.items():
            def run():
                outs[name] = e.hash_fixed(alg, data, msg_len, count, bits, timed=True)
                return e.last_device_ms
            ms = med(run)
            perms = count * permutations(alg, msg_len, bits)
            res.append({"workload": f"{alg} 2^{log2} x {msg_len} B", "kernel": name, "ms": ms,
                        "gb_per_s_hashed": count * msg_len / ms / 1e6,
                        "int_roofline_frac": perms / ms * 1e3 * 4320 / peak})
            print(res[-1], flush=True)
        assert torch.equal(outs["direct (generic)"], outs["TMA-staged"])
        del data, outs
    count = 1 << 22
    e = engines["TMA-staged"]
    lengths = e.generate_lengths(count, 1, 16384, seed_len=2)
    padded = (lengths + 7) // 8 * 8
    offsets = torch.cumsum(padded, 0) - padded
    data = torch.empty(int(padded.sum().item()) + 16, dtype=torch.uint8, device="cuda")
    e.fill_messages(data, offsets, lengths, seed=1)
    nbytes = int(lengths.sum().item())
    perms = int((lengths // 136 + 1).sum().item())
    outs = {}
    for name, eng in engines.items():
        def run():
            outs[name] = eng.hash_batch("sha3_256", data, offsets, lengths, timed=True)
            return eng.last_device_ms
        ms = med(run, reps=3)
        res.append({"workload": "cfg4 sha3_256 2^22 x 1..16 KiB (bucketed)", "kernel": name, "ms": ms,
                    "gb_per_s_hashed": nbytes / ms / 1e6, "int_roofline_frac": perms / ms * 1e3 * 4320 / peak})
        print(res[-1], flush=True)
    assert torch.equal(outs["direct (generic)"], outs["TMA-staged"])
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "staged_vs_direct.json").write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
