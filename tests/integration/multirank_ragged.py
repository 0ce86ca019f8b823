#!/usr/bin/env python3
"""A variable-length batch sharded over the ranks of a process group by cumulative BLOCK count
(sharding.shard_ranges_by_blocks: SURVEY.md 8(e), the plan_partition analogue of
proj/core/src/batch.cpp:46-62 for uneven messages), every rank hashing its contiguous range with
the CUDA path; rank 0 checks the concatenated digests against the unsharded call and a sample
against the CPU oracle, and prints one JSON line.  Launched by tests/test_gpu_multirank.py under
torch.distributed.run (ranks share device 0 on a one-GPU box; gloo group)."""
import json
import os
import pathlib
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = pathlib.Path(__file__).resolve().parent.parent.parent
sys.path.insert(0, str(ROOT))
from oracle.binding import Oracle  # noqa: E402  (test infrastructure)
from paper_1902_05320_b200 import Engine, rate_bytes  # noqa: E402
from paper_1902_05320_b200.sharding import shard_ranges_by_blocks  # noqa: E402


def main():
    algorithm, count = "sha3_256", int(sys.argv[1]) if len(sys.argv) > 1 else 30000
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    rng = np.random.default_rng(4242)                       # the same batch on every rank
    lengths = rng.integers(0, 3000, count).astype(np.uint64)
    lengths[rng.integers(0, count, 20)] = rng.integers(20000, 200000, 20).astype(np.uint64)  # a few heavy ones
    padded = (lengths + np.uint64(7)) // np.uint64(8) * np.uint64(8)
    offsets = (np.cumsum(padded) - padded).astype(np.uint64)
    data = rng.integers(0, 256, int(padded.sum()) + 16, dtype=np.uint8)
    ranges = shard_ranges_by_blocks(lengths, rate_bytes(algorithm), world)
    first, n = ranges[rank]
    engine = Engine(device=0)
    lo = int(offsets[first]) if n else 0
    hi = int(offsets[first + n - 1] + lengths[first + n - 1]) if n else 0
    d_data = torch.from_numpy(data[lo:hi + 16].copy()).cuda()
    d_off = torch.from_numpy((offsets[first:first + n] - np.uint64(lo)).astype(np.int64)).cuda()
    d_len = torch.from_numpy(lengths[first:first + n].astype(np.int64)).cuda()
    mine = engine.hash_batch(algorithm, d_data, d_off, d_len).cpu().numpy() if n else np.zeros((0, 32), np.uint8)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((first, n, mine.tobytes()), gathered, dst=0)
    if rank == 0:
        whole = engine.hash_batch(algorithm, torch.from_numpy(data).cuda(), torch.from_numpy(offsets.astype(np.int64)).cuda(),
                                  torch.from_numpy(lengths.astype(np.int64)).cuda()).cpu().numpy()
        parts = b"".join(g[2] for g in sorted(gathered))
        oracle = Oracle()
        sample = rng.integers(0, count, 64)
        sample_ok = all(oracle.hash_one(1, data[int(offsets[i]):int(offsets[i] + lengths[i])].tobytes())
                        == whole[i].tobytes() for i in sample)
        blocks = lengths // np.uint64(rate_bytes(algorithm)) + np.uint64(1)
        work = [int(blocks[f:f + c].sum()) for f, c in ranges]
        print(json.dumps({"ranks": world, "messages": count, "ranges": ranges, "blocks_per_rank": work,
                          "sharded_equals_unsharded": parts == whole.tobytes(), "oracle_sample_ok": bool(sample_ok)}),
              flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
