"""Multi-GPU host logic: contiguous message ranges per rank, no data-path
collective.

The reference splits a batch into contiguous index ranges and lets one writer
own each output slot (plan_partition, proj/core/src/batch.cpp:46-62;
batch.hpp:61-64).  Across GPUs we do the same one level up: rank g of G owns
messages [g*N/G, (g+1)*N/G) of a fixed-length batch, or -- for variable-length
batches -- a contiguous range balanced by the number of Keccak-f permutations
(block count), which is what the work is proportional to.  Each rank reads and
writes only its own HBM; digests are identical whatever G is because the
synthetic stream is indexed by global message number.
"""
from __future__ import annotations

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """(first, count) of rank's contiguous range; ranges tile [0, total) exactly."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    first = total * rank // world
    return first, total * (rank + 1) // world - first


def shard_ranges_by_blocks(lengths, rate_bytes: int, world: int) -> list[tuple[int, int]]:
    """Contiguous ranges with (nearly) equal sums of floor(len/rate)+1 (permutations)."""
    blocks = np.asarray(lengths, dtype=np.uint64) // np.uint64(rate_bytes) + np.uint64(1)
    csum = np.concatenate([[0], np.cumsum(blocks, dtype=np.uint64)])
    total = int(csum[-1])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(csum, total * r // world, side="left")))
    cuts.append(len(blocks))
    cuts = [min(max(c, cuts[i - 1] if i else 0), len(blocks)) for i, c in enumerate(cuts)]
    return [(cuts[r], cuts[r + 1] - cuts[r]) for r in range(world)]


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the timing rule: a multi-GPU number is the slowest rank's)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_digests(local, total: int, digest_bytes: int):
    """The optional step AFTER the hot path: every rank receives the digests
    of the whole batch, in message order, from the contiguous shards of shard_range().
    `local` is this rank's (count, digest_bytes) uint8 tensor -- on the GPU under NCCL (the
    exchange then runs over NVLink), on the CPU under gloo.  One all_gather of equal-sized
    blocks (shards differ by at most one message; the short ones are padded), then the padding
    is cut out.  Nothing on the data path needs this: digests stay with their shard unless a
    caller wants them in one place."""
    import torch
    import torch.distributed as dist
    local = local.reshape(-1, digest_bytes)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        assert local.shape[0] == total
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    counts = [shard_range(total, r, world)[1] for r in range(world)]
    assert local.shape[0] == counts[rank], "local digests do not match this rank's shard"
    widest = max(counts)
    block = local
    if counts[rank] < widest:
        block = torch.zeros((widest, digest_bytes), dtype=local.dtype, device=local.device)
        block[:counts[rank]] = local
    out = torch.empty((world, widest, digest_bytes), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out.view(-1), block.contiguous().view(-1))
    if min(counts) == widest:
        return out.view(total, digest_bytes)
    return torch.cat([out[r, :counts[r]] for r in range(world)])


def xor_fold_checksum(digest_bytes: np.ndarray) -> int:
    """Order-independent 64-bit checksum of a digest array: XOR of all 8-byte words.
    The XOR over ranks of per-rank values equals the single-GPU value."""
    flat = np.ascontiguousarray(digest_bytes).reshape(-1)
    pad = (-flat.size) % 8
    if pad:
        flat = np.concatenate([flat, np.zeros(pad, dtype=np.uint8)])
    return int(np.bitwise_xor.reduce(flat.view(np.uint64))) if flat.size else 0


def workload_slice(total_bytes: int, message_size: int, first_message: int, count: int,
                   seed: int = 1) -> np.ndarray:
    """Host (numpy) version of the counter-based workload stream: the bytes of messages
    [first_message, first_message+count) of generate_workload(seed, total_bytes, size)
    (proj/tools/sha3cli/workload.cpp:16-47).  Harness only."""
    from .engine import splitmix64_at
    wpm = (message_size + 7) // 8
    stream_seed = (seed ^ (total_bytes * 0x9e3779b97f4a7c15)) & (2**64 - 1)
    n0 = first_message * wpm
    words = splitmix64_at(np.uint64(stream_seed),
                          np.arange(n0 + 1, n0 + count * wpm + 1, dtype=np.uint64))
    full = words.view(np.uint8).reshape(count, wpm * 8)
    return np.ascontiguousarray(full[:, :message_size]).reshape(-1)
