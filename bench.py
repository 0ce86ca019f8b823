#!/usr/bin/env python3
"""bench.py -- the headline benchmark of the batch SHA-3 path.

    python bench.py --gpus N --steps K --warmup W            (N=1 directly,
    python -m torch.distributed.run ... bench.py --gpus N    one rank per GPU for N>1)
    python bench.py --impl reference ...                     (the reference's CPU path)

Workload (BASELINE.json configs[4], the one the metric is quoted on): SHA3-256
over 2^28 x 64-byte messages of the reference's synthetic stream
(proj/tools/sha3cli/workload.cpp:16-47, seed 1), sharded over the N ranks by
contiguous message ranges; no collective on the data path.  One "step" = one
pass of the hot path over the rank's shard, input already resident in HBM,
digests left in HBM.  The total is fixed, so the run is a strong-scaling run.

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

ALGORITHM = "sha3_256"
MSG_LEN = 64
DIGEST_BYTES = 32
INSTR_PER_PERMUTATION = 4320        # 122 LOP3 + 58 SHF per round x 24
METRIC = "SHA3-256 hashes/s on 64-B msg batches"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--log2-messages", type=int, default=28, help="total messages across all GPUs")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = min(steps, 5)")
    ap.add_argument("--cpu-log2-messages", type=int, default=22, help="CPU baseline sample size")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-probe", action="store_true")
    ap.add_argument("--no-dropin", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg1..cfg4 device-time points")
    ap.add_argument("--gather-digests", action="store_true",
                    help="N>1: after the timed region, all-gather the digests to every rank (the optional "
                         "step after the hot path, SURVEY.md 8(e)) and report its time")
    ap.add_argument("--quick-configs", action="store_true", help=argparse.SUPPRESS)
    # validation only (one-GPU box): run N ranks on the SAME device with a gloo process group
    # to exercise the multi-rank code path; numbers from such a run are not benchmark values
    ap.add_argument("--share-gpu", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args()


# --------------------------------------------------------------------------
# clocks: sample nvidia-smi while the timed region runs (B200_PROFILING.md)
class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu_index = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu_index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._pump, daemon=True)
        self.thread.start()

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for name, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        busy = [c for c, p in zip(sm, power) if p > 0.5 * max(power)] if power else sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def host_memory_available():
    """Bytes of host memory this process can still take: MemAvailable, capped by the cgroup
    limit when there is one (0 if unknown)."""
    avail = 0
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                avail = int(line.split()[1]) * 1024
    except OSError:
        pass
    try:
        limit = open("/sys/fs/cgroup/memory.max").read().strip()
        used = int(open("/sys/fs/cgroup/memory.current").read().strip())
        if limit != "max":
            room = max(int(limit) - used, 0)
            avail = min(avail, room) if avail else room
    except (OSError, ValueError):
        pass
    return avail


def measured_peaks():
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        try:
            d = json.loads(path.read_text())
            return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured (MEASURED_PEAKS.json)"
        except (ValueError, KeyError):
            pass
    return 6650.0, 1965.0, "fallback (B200_PROFILING.md)"


def ncu_traffic_per_launch(count_per_launch: int):
    """(dram bytes per launch of the dominant kernel, where the figure comes from): the committed
    `ncu --set full` capture of this command (profiles/roofline_traffic.json, made by
    tools/ncu_traffic.py).  Used as captured when the capture's launch size equals this run's,
    scaled per message otherwise; (None, reason) if there is no capture."""
    path = ROOT / "profiles" / "roofline_traffic.json"
    if not path.exists():
        return None, "no ncu capture committed"
    try:
        d = json.loads(path.read_text())
        if d["messages_per_launch"] == count_per_launch:
            return d["dram_bytes_read_per_launch"] + d["dram_bytes_write_per_launch"], d["source"]
        return (d["dram_bytes_per_message"] * count_per_launch,
                d["source"] + f" scaled from {d['messages_per_launch']} messages per launch")
    except (ValueError, KeyError):
        return None, "profiles/roofline_traffic.json unreadable"


def executed_instr_per_hash(kernel: str):
    """LOP3+SHF instructions one thread EXECUTES per hash in the built kernel, from the SASS
    census (tools/sass_census.py -> profiles/sass_census.json); None if not generated."""
    path = ROOT / "profiles" / "sass_census.json"
    try:
        return json.loads(path.read_text())[kernel]["executed_per_thread"]["LOP3+SHF"]
    except (OSError, ValueError, KeyError):
        return None


# --------------------------------------------------------------------------
def config_points(engine, peak_instr_per_s: float, hbm_peak_gbs: float, quick: bool = False):
    """Device-time points for BASELINE.json configs[0..3] (the headline line is configs[4]):
    median of 5 launches after 2 warm-ups, CUDA events around the kernels on the launching
    stream (cfg.device_ms), inputs resident in HBM and (except cfg1, see its note) larger than
    L2.  `quick` shrinks every batch 64x (the CPU-side contract test of the record shape)."""
    import torch

    from paper_1902_05320_b200 import digest_bytes, permutations, selected_kernel

    shrink = 6 if quick else 0
    points = []

    def record(name, alg, count, msg_bytes, perms, ms, kernel, **extra):
        out_bytes = count * extra["digest_bytes"]
        rate = perms / ms * 1e3
        points.append({"config": name, "algorithm": alg, "messages": count, **extra, "ms": ms,
                       "hashes_per_s": count / ms * 1e3, "gb_per_s_hashed": msg_bytes / ms / 1e6,
                       "perms_per_s": rate, "int_roofline_frac": rate * INSTR_PER_PERMUTATION / peak_instr_per_s,
                       "hbm_gb_per_s": (msg_bytes + out_bytes) / ms / 1e6,
                       "hbm_frac": (msg_bytes + out_bytes) / ms / 1e6 / hbm_peak_gbs, "kernel": kernel})

    def median_ms(run, reps=5, warm=2):
        for _ in range(warm):
            run()
        return statistics.median(run() for _ in range(reps))

    def fixed(name, alg, log2_count, msg_len, bits, back_to_back=0):
        count = 1 << (log2_count - shrink)
        data = engine.generate_workload(count * msg_len, msg_len, seed=1)
        nbytes = digest_bytes(alg, bits)
        out = torch.empty((count, nbytes), dtype=torch.uint8, device="cuda")
        extra = {}
        if back_to_back:
            # sub-millisecond launch: a train of launches between two events
            # on the launching stream, per-launch steady state
            for _ in range(8):
                engine.hash_fixed(alg, data, msg_len, count, bits, out=out)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            trains = []
            for _ in range(3):
                e0.record()
                for _ in range(back_to_back):
                    engine.hash_fixed(alg, data, msg_len, count, bits, out=out)
                e1.record()
                e1.synchronize()
                trains.append(e0.elapsed_time(e1) / back_to_back)
            ms = statistics.median(trains)
            extra = {"launches_per_train": back_to_back,
                     "l2": "working set (%.0f MiB) fits the 126 MB L2: steady-state launches re-read an "
                           "L2-resident input; the kernel is ALU-bound either way" % (count * (msg_len + nbytes) / 2**20)}
        else:
            def run():
                engine.hash_fixed(alg, data, msg_len, count, bits, out=out, timed=True)
                return engine.last_device_ms
            ms = median_ms(run)
        record(name, alg, count, count * msg_len, count * permutations(alg, msg_len, bits), ms,
               selected_kernel(alg, msg_len, bits, count), msg_len=msg_len, xof_bits=bits, digest_bytes=nbytes,
               **extra)

    fixed("cfg1: 2^20 x 64 B", "sha3_256", 20, 64, 0, back_to_back=200 if not quick else 20)
    for alg, msg_len in (("sha3_224", 128), ("sha3_384", 256), ("sha3_512", 1024)):
        fixed("cfg2: 2^24 fixed-length", alg, 24, msg_len, 0)
    for alg, bits in (("shake128", 1024), ("shake256", 4096)):
        fixed("cfg3: 2^24 x 64 B XOF", alg, 24, 64, bits)

    # cfg4: 2^22 messages, lengths uniform 1..16384 (seed_len 2), 8-byte aligned
    # starts, bucketed by block count on the device
    count = 1 << (22 - shrink)
    lengths = engine.generate_lengths(count, 1, 16384, seed_len=2)
    padded = (lengths + 7) // 8 * 8
    offsets = torch.cumsum(padded, 0) - padded
    data = torch.empty(int(padded.sum().item()) + 16, dtype=torch.uint8, device="cuda")
    engine.fill_messages(data, offsets, lengths, seed=1)
    out = torch.empty((count, 32), dtype=torch.uint8, device="cuda")
    msg_bytes = int(lengths.sum().item())
    perms = int((lengths // 136 + 1).sum().item())

    def run():
        engine.hash_batch("sha3_256", data, offsets, lengths, out=out, timed=True)
        return engine.last_device_ms
    ms = median_ms(run, reps=3, warm=1)
    record("cfg4: 2^22 x 1 B..16 KiB", "sha3_256", count, msg_bytes, perms, ms,
           selected_kernel("sha3_256", None, 0, count),
           digest_bytes=32, mean_len=msg_bytes / count, metadata_bytes_per_message=16,
           launches_per_call=engine.last_kernel_launches,
           note="device time of the whole call: bucketing passes (histogram, scan, scatter) + hash kernel")
    del data, out, offsets, lengths, padded
    torch.cuda.empty_cache()

    # Beyond BASELINE.json's configs: few long messages, where the sponge chain's latency is all
    # there is (one warp per message, csrc/kernel_warp.cu) -- next to the same batch with one
    # message per thread.
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import FLAG_NO_WARP_KERNEL
    count, msg_len = (1024, 1 << 20) if not quick else (64, 1 << 16)
    data = engine.generate_workload(count * msg_len, msg_len, seed=1)
    out = torch.empty((count, 32), dtype=torch.uint8, device="cuda")
    per_thread = Engine(device=engine.device, flags=FLAG_NO_WARP_KERNEL)
    times = {}
    for name, eng in (("warp", engine), ("thread", per_thread)):
        def run():
            eng.hash_fixed("sha3_256", data, msg_len, count, out=out, timed=True)
            return eng.last_device_ms
        times[name] = median_ms(run, reps=3, warm=1)
    record("few long messages: 1024 x 1 MiB", "sha3_256", count, count * msg_len,
           count * permutations("sha3_256", msg_len), times["warp"], selected_kernel("sha3_256", msg_len, 0, count),
           msg_len=msg_len, xof_bits=0, digest_bytes=32, ms_one_message_per_thread=times["thread"],
           note="latency-bound (a sponge is sequential per message): the roofline fraction says how much of the "
                "machine 1024 messages can use, not how good the kernel is")
    return points


# --------------------------------------------------------------------------
def cpu_baseline(log2_messages: int, steps: int, warmup: int):
    """The reference's own hash_batch (oracle/_ref, compiled from /root/reference) or,
    where that library does not exist, the C restatement -- on the host cores, on a bounded
    sample of the SAME workload stream.  Median of `steps` runs after `warmup`."""
    from oracle.binding import Oracle, Reference
    count = 1 << log2_messages
    total_bytes = (1 << 28) * MSG_LEN            # the stream of the full workload; we take its head
    oracle = Oracle()
    # head of the full-size stream (same seed derivation as the GPU arm: workload.cpp:34)
    from paper_1902_05320_b200.sharding import workload_slice
    data = workload_slice(total_bytes, MSG_LEN, 0, count, seed=1)
    cores = os.cpu_count() or 1
    variants = {}
    if Reference.available():
        # Both builds of the reference (oracle/Makefile): "as_shipped" = batch.cpp:108 calling
        # hash_one (one allocated digest vector per message, what the source asks for);
        # "hash_into" = the same line hashing into the pre-sized slot (BASELINE.md section 3's
        # one-line change, made by oracle/ref_prelude.hpp).  The FASTER one is the baseline.
        seq_rate = None
        for name, hash_into in (("as_shipped", False), ("hash_into", True)):
            if not Reference.available(hash_into):
                continue
            ref = Reference(hash_into)
            cores = ref.hardware_workers()
            batch = Reference.Batch(ref, 1, data, MSG_LEN, count)
            runs = [batch.run(parallel=True, workers=0) for _ in range(warmup + steps)][warmup:]
            batch.close()
            variants[name] = runs
            if seq_rate is None:
                seq_count = min(count, 1 << 20)
                seq_batch = Reference.Batch(ref, 1, data[:seq_count * MSG_LEN], MSG_LEN, seq_count)
                seq = [seq_batch.run(parallel=False) for _ in range(3)]
                seq_batch.close()
                seq_rate = seq_count / statistics.median(seq)
        best = min(variants, key=lambda k: statistics.median(variants[k]))
        times = variants[best]
        kind = "reference"
    else:
        best = "oracle port"
        t = []
        for _ in range(warmup + steps):
            t0 = time.perf_counter()
            oracle.hash_batch(1, data, fixed_len=MSG_LEN, count=count, workers=cores)
            t.append(time.perf_counter() - t0)
        times = t[warmup:]
        kind = "port"
        t0 = time.perf_counter()
        oracle.hash_batch(1, data, fixed_len=MSG_LEN, count=min(count, 1 << 20), workers=1)
        seq_rate = min(count, 1 << 20) / (time.perf_counter() - t0)
    med = statistics.median(times)
    return {"value": count / med, "unit": "hashes/s", "cores": cores, "kind": kind,
            "sample": f"first 2^{log2_messages} messages of the same stream, hash_batch "
                      f"Backend::parallel workers={cores}, median of {steps} runs after {warmup} warm-up",
            "build": best,
            "builds_hashes_per_s": {k: count / statistics.median(v) for k, v in variants.items()},
            "ms_per_run": med * 1e3, "sequential_1core_hashes_per_s": seq_rate}, med


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    base, med = cpu_baseline(args.cpu_log2_messages, args.steps, args.warmup)
    count = 1 << args.cpu_log2_messages
    line = {
        "impl": "reference", "metric": METRIC, "value": base["value"], "unit": "hashes/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": med * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (reference generate_workload stream, seed 1)",
        "config": {"workload": f"SHA3-256 over 2^{args.log2_messages} x 64-byte messages (BASELINE.json "
                               f"configs[4]); each step a bounded sample of 2^{args.cpu_log2_messages} "
                               "messages on the host cores", "messages_per_step": count,
                   "message_bytes": MSG_LEN},
        "gb_per_s_hashed": base["value"] * MSG_LEN / 1e9,
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "hashes/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def dropin_cpp_wall(log2_messages: int = 24):
    """The same metric one level further out: the reference's own C++ interface,
    sha3::hash_batch on vector<vector<uint8_t>> (proj/core/include/sha3/batch.hpp:23-65), served by
    the drop-in adapter -- pack + H2D + kernels + D2H + unpack all inside the call, wall clock.
    Measured by tests/cpp/dropin_wall (tests/integration/dropin_wall.cpp) in its own process;
    None if that binary was not built."""
    exe = ROOT / "tests" / "cpp" / "dropin_wall"
    if not exe.exists():
        return None
    try:
        out = subprocess.run([str(exe), str(log2_messages), str(MSG_LEN), "5", "none"], capture_output=True,
                             text=True, timeout=300, cwd=str(ROOT))
        rec = json.loads(out.stdout)
        d = rec["b200_dropin"]
        return {"value": d["hashes_per_s"], "unit": "hashes/s", "messages_per_call": rec["count"],
                "wall_ms_per_call": d["wall_s"] * 1e3, "host_threads": rec["host_threads"],
                "stages_ms": {k: d[k] * 1e3 for k in ("resize_s", "device_calls_s", "pack_cpu_s", "unpack_cpu_s")},
                "note": "sha3::b200::hash_batch(HashBatch) -> BatchResult on vector<vector<uint8_t>>, "
                        "median of 5 calls; pack/unpack CPU times are summed over the host threads"}
    except (OSError, ValueError, KeyError, subprocess.SubprocessError):
        return None


# --------------------------------------------------------------------------
def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    from paper_1902_05320_b200 import Engine, library_info

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with torch.distributed.run")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU fallback)")
    if args.share_gpu:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    reduce_device = "cpu" if args.share_gpu else "cuda"
    if world > 1:
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    from paper_1902_05320_b200.sharding import max_over_ranks as _max_over_ranks, shard_range

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        return _max_over_ranks(x, device=reduce_device)

    total = 1 << args.log2_messages
    total_bytes = total * MSG_LEN
    # contiguous message range per rank (plan_partition analogue, batch.cpp:46-62)
    first, count = shard_range(total, rank, world)

    engine = Engine(device=local_rank)
    data = engine.generate_workload(total_bytes, MSG_LEN, seed=1, first_message=first, count=count)
    digests = torch.empty((count, DIGEST_BYTES), dtype=torch.uint8, device="cuda")

    warmup = max(args.warmup, 3)      # timing rule: at least three untimed steps
    for _ in range(warmup):
        engine.hash_fixed(ALGORITHM, data, MSG_LEN, count, out=digests)
    sampler = ClockSampler(local_rank)
    if rank == 0:
        sampler.start()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches_before = engine.total_kernel_launches
    barrier()
    start.record()
    for _ in range(args.steps):
        engine.hash_fixed(ALGORITHM, data, MSG_LEN, count, out=digests)
    stop.record()
    barrier()
    clocks = sampler.stop() if rank == 0 else None
    seconds = max_over_ranks(start.elapsed_time(stop) * 1e-3)
    launches = engine.total_kernel_launches - launches_before
    if world > 1:  # every rank's kernels count: sum over ranks
        n = torch.tensor([launches], dtype=torch.int64, device=reduce_device)
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
        launches = int(n.item())
    value = total * args.steps / seconds

    # checksum of the digests: sum of their 64-bit words mod 2^64 -- proves the timed
    # kernels did the work, and is the same number for every N (sum over ranks)
    t = digests.view(torch.int64).sum().reshape(1).to(reduce_device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    checksum = int(t.item()) & (2**64 - 1)

    # ---- optional: digests of the whole batch on every rank (NCCL all-gather over NVLink; the
    # hot path never needs it -- digests stay with their shard unless requested) ----------
    gather = None
    if args.gather_digests and world > 1:
        from paper_1902_05320_b200.sharding import gather_digests
        local = digests.cpu() if args.share_gpu else digests
        barrier()
        t0 = time.perf_counter()
        everything = gather_digests(local, total, DIGEST_BYTES)
        torch.cuda.synchronize()
        gather_seconds = max_over_ranks(time.perf_counter() - t0)
        gathered_sum = int(everything.view(torch.int64).sum().item()) & (2**64 - 1)
        gather = {"ms": gather_seconds * 1e3, "bytes_per_rank": total * DIGEST_BYTES,
                  "checksum_matches": gathered_sum == checksum,
                  "backend": "gloo (host tensors; validation only)" if args.share_gpu else "nccl"}
        del everything, local

    # ---- end to end through the host-buffer C entry (pinned host memory) -----------
    e2e = None
    if not args.no_e2e:
        # Host staging for the whole shard (16 GiB + 8 GiB at N=1).  If the box cannot pin that
        # much, halve the end-to-end batch until it can and say so in the line.
        e2e_count = count
        avail = host_memory_available()
        while e2e_count > 1 and avail and e2e_count * (MSG_LEN + DIGEST_BYTES) * world > 0.6 * avail:
            e2e_count //= 2
        while True:
            try:
                host_in = torch.empty(e2e_count * MSG_LEN, dtype=torch.uint8).pin_memory()
                host_out = torch.empty(e2e_count * DIGEST_BYTES, dtype=torch.uint8).pin_memory()
                break
            except RuntimeError:
                if e2e_count <= (1 << 20):
                    raise
                e2e_count //= 2
        host_in.copy_(data[:e2e_count * MSG_LEN])
        torch.cuda.synchronize()
        e2e_steps = args.e2e_steps or min(args.steps, 5)
        engine.hash_fixed_ptr(ALGORITHM, host_in.data_ptr(), MSG_LEN, e2e_count, host_out.data_ptr())
        barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            engine.hash_fixed_ptr(ALGORITHM, host_in.data_ptr(), MSG_LEN, e2e_count, host_out.data_ptr())
        torch.cuda.synchronize()
        e2e_seconds = max_over_ranks(time.perf_counter() - t0)
        same = bool(torch.equal(host_out.view(e2e_count, DIGEST_BYTES)[:4096], digests[:4096].cpu()))
        # what bounds e2e: the PCIe link.  A plain pinned H2D copy of the same buffer, alone
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        data[:e2e_count * MSG_LEN].copy_(host_in, non_blocking=True)
        torch.cuda.synchronize()
        plain_h2d_gbs = e2e_count * MSG_LEN / (time.perf_counter() - t0) / 1e9
        # ... and the ceiling of the call's shape: the same input and output buffers copied BOTH
        # ways at once on two streams, no hashing (tools/microbench/pcie_duplex.cu is the
        # stand-alone form).  H2D runs slower under opposite traffic than alone.
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        duplex_seconds = None
        for _ in range(2):          # the faster of two passes
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with torch.cuda.stream(s_in):
                data[:e2e_count * MSG_LEN].copy_(host_in, non_blocking=True)
            with torch.cuda.stream(s_out):
                host_out.copy_(digests.view(-1)[:e2e_count * DIGEST_BYTES], non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            duplex_seconds = dt if duplex_seconds is None else min(duplex_seconds, dt)
        duplex_seconds = max_over_ranks(duplex_seconds)
        e2e_total = e2e_count * world if e2e_count != count else total
        e2e = {"value": e2e_total * e2e_steps / e2e_seconds, "unit": "hashes/s",
               "h2d_bytes_per_step": e2e_total * MSG_LEN, "d2h_bytes_per_step": e2e_total * DIGEST_BYTES,
               "messages_per_step": e2e_total,
               "steps": e2e_steps, "ms_per_step": e2e_seconds / e2e_steps * 1e3,
               "digests_match_device_path": same,
               "pcie": {"h2d_gb_per_s_inside_pipeline": e2e_count * MSG_LEN * e2e_steps / e2e_seconds / 1e9,
                        "d2h_gb_per_s_inside_pipeline": e2e_count * DIGEST_BYTES * e2e_steps / e2e_seconds / 1e9,
                        "h2d_gb_per_s_plain_pinned_copy": plain_h2d_gbs,
                        "duplex_plain_copies": {
                            "ms": duplex_seconds * 1e3,
                            "h2d_gb_per_s": e2e_count * MSG_LEN / duplex_seconds / 1e9,
                            "d2h_gb_per_s": e2e_count * DIGEST_BYTES / duplex_seconds / 1e9,
                            "note": "input and output buffers of one step copied both ways at once, no "
                                    "hashing: the floor for one e2e step on this link"},
                        "e2e_step_over_duplex_copies": e2e_seconds / e2e_steps / duplex_seconds,
                        "note": "per rank; e2e is bound by the host link, not by the kernel"},
               "note": "b200sha3_hash_fixed on pinned host buffers: chunked H2D / kernel / D2H "
                       "pipeline inside the call; wall clock, max over ranks"}
        del host_in, host_out

    if rank == 0:
        hbm_peak, sm_max_mhz, peak_src = measured_peaks()
        perms_per_s = value                      # one Keccak-f[1600] per 64-byte SHA3-256 message
        achieved = perms_per_s / world * INSTR_PER_PERMUTATION / 1e12   # per GPU
        nominal_peak = 148 * 64 * sm_max_mhz * 1e6 / 1e12
        probe = None
        if not args.no_probe:
            rate, hz = engine.probe_pipe(2)      # LOP3+SHF 2:1, the Keccak ALU mix
            probe = {"instr_per_s": rate, "sm_hz": hz}
        peak = probe["instr_per_s"] / 1e12 if probe else nominal_peak
        per_launch = count
        kernel_name = "hash_oneblock_kernel<17, 8, 8, 23, 0u>"
        executed = executed_instr_per_hash(kernel_name)
        traffic, traffic_source = ncu_traffic_per_launch(per_launch)
        line = {
            "metric": METRIC, "value": value, "unit": "hashes/s", "n_gpus": world,
            "steps": args.steps, "warmup": warmup, "ms_per_step": seconds / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (reference generate_workload stream, seed 1, generated on device)",
            **({"validation_only": "ranks share one GPU (gloo); not a benchmark value"} if args.share_gpu else {}),
            "config": {"workload": f"SHA3-256 over 2^{args.log2_messages} x 64-byte messages sharded "
                                   f"over {world} GPU(s) by contiguous ranges (BASELINE.json configs[4])",
                       "messages_total": total, "messages_per_gpu": count, "message_bytes": MSG_LEN,
                       "l2_policy": "inputs larger than L2 (%.1f GiB per GPU per step)" % (count * MSG_LEN / 2**30),
                       "kernel": kernel_name + " (UNROLL 23 = peeled 1 + 7x3 + 2 rounds, ALU only)"},
            "gb_per_s_hashed": value * MSG_LEN / 1e9,
            "gpu_launches": launches,
            "library": library_info(),
            "digest_checksum": f"{checksum:016x}",
            "clocks": clocks,
            "roofline": {
                "bound": "int_alu",
                "achieved": achieved, "peak": peak, "unit": "Tinstr/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": traffic_source,
                "algorithmic_bytes_per_launch": per_launch * (MSG_LEN + DIGEST_BYTES),
                "instr_per_hash_contract": INSTR_PER_PERMUTATION,
                "instr_executed_per_hash": executed,
                "frac_executed": (achieved * executed / INSTR_PER_PERMUTATION / peak) if executed else None,
                "note": "per GPU; achieved = permutations/s x 4320 LOP3+SHF thread-instructions "
                        "(SURVEY.md 8(d)'s contract figure); peak = LOP3+SHF issue rate measured in this "
                        "run by b200sha3_probe_pipe" + ("" if probe else " [probe skipped: nominal]") +
                        ".  frac can read above 1 because the built kernel executes fewer than 4320 "
                        "(instr_executed_per_hash, from the SASS census: ptxas removes dead work in "
                        "rounds 0 and 23); frac_executed is the share of the pipe's issue slots the "
                        "kernel actually fills",
                "peak_nominal": nominal_peak,
                "probe_sm_mhz": probe["sm_hz"] / 1e6 if probe else None,
            },
            "roofline_hbm": {
                "bound": "hbm", "achieved": value / world * (MSG_LEN + DIGEST_BYTES) / 1e9,
                "peak": hbm_peak, "unit": "GB/s",
                "frac": value / world * (MSG_LEN + DIGEST_BYTES) / 1e9 / hbm_peak,
                "peak_source": peak_src,
                "note": "secondary: 96 algorithmic bytes per message; not the binding roofline",
            },
        }
        if e2e:
            line["e2e"] = e2e
        if gather:
            line["digest_gather"] = gather
        if world == 1 and not args.no_dropin:
            dropin = dropin_cpp_wall()
            if dropin:
                line["dropin_cpp"] = dropin
        if world == 1 and not args.no_configs:
            del data, digests
            torch.cuda.empty_cache()
            line["configs"] = config_points(engine, peak * 1e12, hbm_peak, quick=args.quick_configs)
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"], _ = cpu_baseline(args.cpu_log2_messages, 5, 2)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
