"""Multi-GPU host logic on CPU: shard planning, stream slicing, and a
world_size-2 gloo run in which each rank hashes its shard (with the oracle --
there is no GPU here) and rank 0 checks the gathered digests against the
unsharded run."""
import os
import socket

import numpy as np
import pytest

from paper_1902_05320_b200.sharding import (shard_range, shard_ranges_by_blocks, workload_slice,
                                            xor_fold_checksum)


def test_shard_ranges_tile_the_batch():
    for total in (0, 1, 7, 1000, 2**28, 2**28 + 5):
        for world in (1, 2, 3, 4, 8):
            expect = 0
            for rank in range(world):
                first, count = shard_range(total, rank, world)
                assert first == expect and count >= 0
                expect += count
            assert expect == total
    assert shard_range(2**28, 3, 8) == (3 * 2**25, 2**25)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_block_balanced_ranges():
    rng = np.random.default_rng(1)
    lengths = rng.integers(1, 16385, 100_000)
    for world in (1, 2, 4, 8):
        ranges = shard_ranges_by_blocks(lengths, 136, world)
        assert ranges[0][0] == 0 and sum(c for _, c in ranges) == len(lengths)
        for (f0, c0), (f1, _) in zip(ranges, ranges[1:]):
            assert f0 + c0 == f1
        work = [int((lengths[f:f + c] // 136 + 1).sum()) for f, c in ranges]
        assert max(work) - min(work) <= 2 * 121          # within one max-size message or two


def test_workload_slice_matches_the_oracle_stream(oracle):
    total_bytes = 1 << 16
    for size in (64, 10, 137):
        whole = oracle.generate_workload(total_bytes, size, seed=1)
        count = total_bytes // size
        for first, n in ((0, 5), (17, 100), (count - 3, 3)):
            part = workload_slice(total_bytes, size, first, n, seed=1)
            assert (part == whole[first * size:(first + n) * size]).all()


def test_checksum_is_shard_invariant():
    rng = np.random.default_rng(2)
    d = rng.integers(0, 256, (1000, 32), dtype=np.uint8)
    whole = xor_fold_checksum(d)
    assert whole == xor_fold_checksum(d[:400]) ^ xor_fold_checksum(d[400:])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, total, out_queue):
    import torch
    import torch.distributed as dist
    from oracle.binding import Oracle
    from paper_1902_05320_b200.sharding import max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = shard_range(total, rank, world)
    data = workload_slice(total * 64, 64, first, count, seed=1)
    digests = Oracle().hash_batch(1, data, fixed_len=64, count=count)
    # timing rule: the slowest rank's time is the job's time
    slowest = max_over_ranks(float(rank + 1))
    gathered = [None] * world
    dist.all_gather_object(gathered, (first, count, xor_fold_checksum(digests), digests[:2].tobytes()))
    if rank == 0:
        out_queue.put((slowest, gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_run_matches_single_rank(oracle):
    import torch.multiprocessing as mp
    total, world = 20_000, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, total, q)) for r in range(world)]
    [p.start() for p in procs]
    slowest, gathered = q.get(timeout=120)
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    assert slowest == float(world)
    whole = oracle.hash_batch(1, oracle.generate_workload(total * 64, 64, seed=1), fixed_len=64, count=total)
    check = 0
    for first, count, checksum, head in gathered:
        assert head == whole[first:first + 2].tobytes()
        check ^= checksum
    assert check == xor_fold_checksum(whole)
    assert [g[:2] for g in gathered] == [shard_range(total, r, world) for r in range(world)]


def _gather_main(rank, world, port, total, out_queue):
    import torch
    import torch.distributed as dist
    from oracle.binding import Oracle
    from paper_1902_05320_b200.sharding import gather_digests
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    first, count = shard_range(total, rank, world)
    data = workload_slice(total * 64, 64, first, count, seed=1)
    local = torch.from_numpy(Oracle().hash_batch(1, data, fixed_len=64, count=count).reshape(count, 32).copy())
    everything = gather_digests(local, total, 32)
    out_queue.put((rank, everything.numpy().tobytes()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total,world", [(20_001, 2), (1_000, 3)])
def test_gathered_digests_are_the_unsharded_result(oracle, total, world):
    """After-the-fact digest gather (optional): every rank ends up with the
    digests of the whole batch in message order, uneven shards included."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_main, args=(r, world, port, total, q)) for r in range(world)]
    [p.start() for p in procs]
    got = dict(q.get(timeout=120) for _ in range(world))
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    whole = oracle.hash_batch(1, oracle.generate_workload(total * 64, 64, seed=1), fixed_len=64, count=total)
    for rank in range(world):
        assert got[rank] == whole.tobytes()


def test_shard_properties_hypothesis():
    """Property form of the partition tests of proj/tests/test_batch.cpp:51-70: ranges are
    contiguous, disjoint and cover the batch, for any batch shape and GPU count."""
    from hypothesis import given, settings, strategies as st

    @settings(max_examples=200, deadline=None)
    @given(st.integers(0, 10**12), st.integers(1, 16))
    def fixed(total, world):
        pos = 0
        sizes = []
        for rank in range(world):
            first, count = shard_range(total, rank, world)
            assert first == pos and count >= 0
            pos += count
            sizes.append(count)
        assert pos == total and max(sizes) - min(sizes) <= 1

    @settings(max_examples=100, deadline=None)
    @given(st.lists(st.integers(0, 20000), min_size=0, max_size=300), st.integers(1, 8),
           st.sampled_from([72, 104, 136, 144, 168]))
    def ragged(lengths, world, rate):
        ranges = shard_ranges_by_blocks(np.array(lengths, dtype=np.uint64), rate, world)
        assert len(ranges) == world
        pos = 0
        for first, count in ranges:
            assert first == pos and count >= 0
            pos += count
        assert pos == len(lengths)
        if lengths:
            blocks = np.array(lengths) // rate + 1
            work = [int(blocks[f:f + c].sum()) for f, c in ranges]
            assert max(work) <= int(blocks.sum()) / world + int(blocks.max()) + 1

    fixed()
    ragged()
