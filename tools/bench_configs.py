#!/usr/bin/env python3
"""Device-time measurements of every BASELINE.json config on one B200 (the
headline bench.py line covers configs[4]; this fills in the rest).  Writes
gpurun_out/configs.json.  Median of 5 timed runs after 2 warm-ups, CUDA events
around the kernels (cfg.device_ms), inputs resident in HBM and larger than L2
unless noted."""
import json
import pathlib
import statistics
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1902_05320_b200 import Engine, digest_bytes, permutations, rate_bytes  # noqa: E402
from paper_1902_05320_b200.engine import FLAG_NO_BUCKETING  # noqa: E402

INSTR = 4320
RESULTS = []


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        ms.append(fn())
    return statistics.median(ms)


def record(name, alg, count, msg_bytes_total, perms_total, ms, peak, extra=None):
    out_bytes = count * extra.pop("digest_bytes")
    rec = {"config": name, "algorithm": alg, "messages": count, "ms": ms,
           "hashes_per_s": count / ms * 1e3, "gb_per_s_hashed": msg_bytes_total / ms / 1e6,
           "perms_per_s": perms_total / ms * 1e3,
           "int_roofline_frac": perms_total / ms * 1e3 * INSTR / peak,
           "hbm_gb_per_s": (msg_bytes_total + out_bytes) / ms / 1e6}
    rec.update(extra or {})
    RESULTS.append(rec)
    print(json.dumps(rec), flush=True)


def fixed(engine, name, alg, log2_count, msg_len, bits, peak):
    count = 1 << log2_count
    data = engine.generate_workload(count * msg_len, msg_len, seed=1)
    out = torch.empty((count, digest_bytes(alg, bits)), dtype=torch.uint8, device="cuda")

    def run():
        engine.hash_fixed(alg, data, msg_len, count, bits, out=out, timed=True)
        return engine.last_device_ms
    ms = timed(run)
    record(name, alg, count, count * msg_len, count * permutations(alg, msg_len, bits), ms, peak,
           {"msg_len": msg_len, "xof_bits": bits, "digest_bytes": digest_bytes(alg, bits)})
    del data, out


def main():
    which = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4"]
    e = Engine()
    peak, hz = e.probe_pipe(2)
    print(f"ALU peak {peak/1e12:.2f} Tinstr/s at {hz/1e6:.0f} MHz", flush=True)
    if "cfg1" in which:
        fixed(e, "cfg1 2^20 x 64B (fits L2)", "sha3_256", 20, 64, 0, peak)
    if "cfg2" in which:
        for alg in ("sha3_224", "sha3_384", "sha3_512"):
            for msg_len in (32, 64, 128, 256, 512, 1024):
                fixed(e, "cfg2 2^24 fixed", alg, 24, msg_len, 0, peak)
    if "cfg3" in which:
        for alg in ("shake128", "shake256"):
            for bits in (256, 512, 1024, 2048, 4096):
                fixed(e, "cfg3 2^24 x 64B XOF", alg, 24, 64, bits, peak)
    if "cfg4" in which:
        count = 1 << (int(sys.argv[sys.argv.index("--cfg4-log2") + 1]) if "--cfg4-log2" in sys.argv else 22)
        lengths = e.generate_lengths(count, 1, 16384, seed_len=2)
        padded = (lengths + 7) // 8 * 8
        offsets = torch.cumsum(padded, 0) - padded
        total = int(padded.sum().item())
        data = torch.empty(total + 16, dtype=torch.uint8, device="cuda")
        e.fill_messages(data, offsets, lengths, seed=1)
        out = torch.empty((count, 32), dtype=torch.uint8, device="cuda")
        msg_bytes = int(lengths.sum().item())
        perms = int((lengths // 136 + 1).sum().item())
        from paper_1902_05320_b200.engine import KERNEL_STAGED
        for label, eng in (("bucketed", e), ("input order (no bucketing)", Engine(flags=FLAG_NO_BUCKETING)),
                           ("bucketed, TMA-staged kernel", Engine(kernel=KERNEL_STAGED))):
            def run():
                eng.hash_batch("sha3_256", data, offsets, lengths, out=out, timed=True)
                return eng.last_device_ms
            ms = timed(run, reps=3, warm=1)
            record(f"cfg4 2^{count.bit_length()-1} x 1..16KiB, {label}", "sha3_256", count, msg_bytes, perms,
                   ms, peak, {"digest_bytes": 32, "mean_len": msg_bytes / count})
    out_dir = ROOT / "gpurun_out"
    out_dir.mkdir(exist_ok=True)
    (out_dir / "configs.json").write_text(json.dumps({"alu_peak_instr_per_s": peak, "sm_hz": hz,
                                                      "results": RESULTS}, indent=1))


if __name__ == "__main__":
    main()
