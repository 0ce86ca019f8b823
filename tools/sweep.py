#!/usr/bin/env python3
"""GPU-box experiment driver: pipe probes + timing of every kernel variant on
the headline workload.  Writes gpurun_out/sweep.json.  Not part of the product."""
import json
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1902_05320_b200 import Engine  # noqa: E402
from paper_1902_05320_b200.engine import KERNEL_GENERIC, KERNEL_ONEBLOCK  # noqa: E402

MIXES = ["LOP3", "SHF", "LOP3+SHF 2:1", "IMAD", "IMAD.WIDE+IMAD", "IMAD.HI", "LOP3+IMAD 1:1",
         "LOP3+(IMAD.WIDE+IMAD)", "LOP3+IMAD.HI 1:1", "keccak flavour-2 mix",
         "pool LOP3", "pool LOP3+IMAD 1:1", "pool LOP3+IMAD 3:1", "pool LOP3+IMAD(1reg) 3:1",
         "pool LOP3+IMAD.HI 3:1", "pool LOP3+SHF 2:1"]


def time_hash(engine, dev, count, reps=5, msg_len=64, alg="sha3_256", bits=0):
    out = engine.hash_fixed(alg, dev, msg_len, count, bits)
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        engine.hash_fixed(alg, dev, msg_len, count, bits, out=out, timed=True)
        ms = engine.last_device_ms
        best = ms if best is None else min(best, ms)
    return best


def main():
    out_dir = ROOT / "gpurun_out"
    out_dir.mkdir(exist_ok=True)
    res = {"device": torch.cuda.get_device_name(0), "probe": {}, "variants": []}
    e = Engine()
    for mix, name in enumerate(MIXES):
        rate, hz = e.probe_pipe(mix)
        res["probe"][name] = {"instr_per_s": rate, "sm_hz": hz,
                              "instr_per_clk_per_sm": rate / hz / 148 if hz else None}
        print(f"probe {name:28s} {rate/1e12:8.3f} Tinstr/s  clk {hz/1e6:7.1f} MHz  "
              f"{rate/hz/148 if hz else 0:6.1f} /clk/SM", flush=True)
    count = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 24)
    dev = e.generate_workload(count * 64, 64, seed=1)
    ref = Engine(kernel=KERNEL_GENERIC).hash_fixed("sha3_256", dev, 64, count)
    for kernel, kname, unrolls in ((KERNEL_ONEBLOCK, "oneblock", (2, 11, 20, 21, 22, 23, 24)), (KERNEL_GENERIC, "generic", (2,))):
        for unroll in unrolls:
            for preset in (0,):
                for threads in ((64, 128, 256) if preset == 0 else (128,)):
                    eng = Engine(kernel=kernel, unroll=unroll, fma_preset=preset, block_threads=threads)
                    ms = time_hash(eng, dev, count)
                    ok = bool(torch.equal(eng.hash_fixed("sha3_256", dev, 64, count), ref))
                    rec = {"kernel": kname, "unroll": unroll, "fma_preset": preset, "threads": threads,
                           "ms": ms, "ghash_per_s": count / ms / 1e6, "ok": ok}
                    res["variants"].append(rec)
                    print(rec, flush=True)
    from paper_1902_05320_b200.engine import KERNEL_LANESPLIT
    eng = Engine(kernel=KERNEL_LANESPLIT)
    ms = time_hash(eng, dev, count, reps=3)
    ok = bool(torch.equal(eng.hash_fixed("sha3_256", dev, 64, count), ref))
    rec = {"kernel": "lanesplit", "unroll": 1, "fma_preset": 0, "threads": 128, "ms": ms,
           "ghash_per_s": count / ms / 1e6, "ok": ok}
    res["variants"].append(rec)
    print(rec, flush=True)
    (out_dir / "sweep.json").write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
