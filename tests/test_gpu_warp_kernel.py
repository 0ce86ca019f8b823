"""The warp-per-state kernel (csrc/kernel_warp.cu: one message per warp, the 25 lanes of
permute_1600 -- proj/core/src/keccak.cpp:245-277 -- spread over 25 threads): bit-exact
against the oracle, the reference's vectors and hashlib, forced and as KERNEL_AUTO picks it
for batches of few multi-block messages."""
import hashlib

import numpy as np
import pytest

from conftest import all_kat_files, load_kat_file, xof_bits_for
from test_gpu_parity import device_digests, to_device

pytestmark = pytest.mark.gpu

HASHLIB = ["sha3_224", "sha3_256", "sha3_384", "sha3_512", "shake_128", "shake_256"]


@pytest.fixture(scope="module")
def warp_engine():
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import KERNEL_WARP
    return Engine(kernel=KERNEL_WARP)


def by_hashlib(algorithm, msg, bits=0):
    h = hashlib.new(HASHLIB[algorithm], bytes(msg))
    return h.digest((bits + 7) // 8) if algorithm >= 4 else h.digest()


@pytest.mark.parametrize("path", all_kat_files(), ids=lambda p: p.stem)
def test_reference_vectors(warp_engine, path):
    """All 892 .rsp vectors, one warp per vector, at three packings (odd starts included)."""
    algorithm, out_bits, vectors = load_kat_file(path)
    bits = xof_bits_for(algorithm, out_bits)
    msgs = [m for m, _ in vectors]
    for align, lead in ((1, 0), (8, 0), (4, 0), (1, 5)):
        got = device_digests(warp_engine, algorithm, msgs, bits, align, lead)
        for row, (_, md) in zip(got, vectors):
            assert row.tobytes() == md


@pytest.mark.parametrize("algorithm", range(6))
def test_block_boundary_lengths(warp_engine, oracle, algorithm):
    """Every length around one, two and three rate blocks (R-1 puts both pad bits in one byte,
    sponge.cpp:122-125), XOF output of 2.5 blocks with an odd bit count."""
    rate = oracle.rate_bytes(algorithm)
    bits = (20 * rate + 3) if algorithm >= 4 else 0
    rng = np.random.default_rng(40 + algorithm)
    lengths = [k * rate + d for k in (0, 1, 2, 3) for d in range(-9, 10) if k * rate + d >= 0] + list(range(0, 20))
    msgs = [rng.integers(0, 256, n, dtype=np.uint8).tobytes() for n in lengths]
    for align in (1, 8):
        got = device_digests(warp_engine, algorithm, msgs, bits, align)
        for row, m in zip(got, msgs):
            assert row.tobytes() == oracle.hash_one(algorithm, m, bits)


@pytest.mark.parametrize("algorithm,msg_len,bits", [(1, 64, 0), (1, 136, 0), (1, 4096, 0), (0, 1000, 0), (2, 777, 0),
                                                    (3, 72 * 5, 0), (4, 64, 4096), (5, 500, 1031), (4, 1, 8)])
def test_fixed_length_entry(warp_engine, oracle, algorithm, msg_len, bits):
    """Equal-length batches through b200sha3_hash_fixed_device, more messages than the
    AUTO threshold (the grid is one block per message)."""
    import torch
    count = 5003
    host = oracle.generate_workload(count * msg_len, msg_len, seed=5)
    expect = oracle.hash_batch(algorithm, host, fixed_len=msg_len, count=count, xof_bits=bits, workers=8)
    got = warp_engine.hash_fixed(algorithm, torch.from_numpy(host).cuda(), msg_len, count, bits)
    assert (got.cpu().numpy() == expect).all()
    assert warp_engine.last_kernel_launches == 1


def test_long_messages_vs_hashlib(warp_engine):
    """The shape the kernel exists for: few long messages (here 48 x ~1 MiB, ragged)."""
    rng = np.random.default_rng(8)
    msgs = [rng.integers(0, 256, (1 << 20) - 37 * i, dtype=np.uint8).tobytes() for i in range(48)]
    for algorithm, bits in ((1, 0), (3, 0), (4, 2048)):
        got = device_digests(warp_engine, algorithm, msgs, bits, align=8)
        for row, m in zip(got, msgs):
            assert row.tobytes() == by_hashlib(algorithm, m, bits)


def test_auto_picks_it_for_small_multiblock_batches(oracle):
    """KERNEL_AUTO: a batch of few messages is one launch of the warp kernel (no bucketing
    passes); the same batch with the kernel switched off takes the classification + bucketing +
    hash launches; both give the oracle's digests.  Single-block equal-length batches keep
    the one-block kernel however few the messages."""
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import FLAG_NO_WARP_KERNEL
    rng = oracle.test_rng(53)
    msgs = [rng.random_bytes(rng.below(2000)) for _ in range(700)]
    expect = [oracle.hash_one(1, m) for m in msgs]
    auto, plain = Engine(), Engine(flags=FLAG_NO_WARP_KERNEL)
    got = device_digests(auto, 1, msgs)
    assert [r.tobytes() for r in got] == expect and auto.last_kernel_launches == 1
    got = device_digests(plain, 1, msgs)
    assert [r.tobytes() for r in got] == expect and plain.last_kernel_launches == 3   # histogram, scatter, hash
    # host entry (the drop-in's path) as well
    assert auto.hash_messages(1, msgs) == expect and plain.hash_messages(1, msgs) == expect
    # equal-length: multi-block -> warp kernel, same digests as the generic kernel
    host = oracle.generate_workload(1000 * 4096, 4096, seed=3)
    dev = torch.from_numpy(host).cuda()
    a = auto.hash_fixed("sha3_512", dev, 4096, 1000)
    b = plain.hash_fixed("sha3_512", dev, 4096, 1000)
    assert torch.equal(a, b)
    assert (a.cpu().numpy() == oracle.hash_batch(3, host, fixed_len=4096, count=1000, workers=8)).all()


def test_empty_messages_and_one_message(warp_engine, oracle):
    for algorithm in range(6):
        bits = 328 if algorithm >= 4 else 0
        msgs = [b"", b"", b"\x00", b""]
        got = device_digests(warp_engine, algorithm, msgs, bits)
        assert [r.tobytes() for r in got] == [oracle.hash_one(algorithm, m, bits) for m in msgs]
        got = device_digests(warp_engine, algorithm, [b"abc"], bits)
        assert got[0].tobytes() == oracle.hash_one(algorithm, b"abc", bits)


@pytest.mark.parametrize("path", all_kat_files()[::3], ids=lambda p: p.stem)
def test_pair_split_kernel(oracle, path):
    """The pair-split comparison kernel (csrc/kernel_pair.cu: low / high halves of every lane in
    two threads, one shuffle per rotation) gives the same digests: reference vectors at odd and
    aligned packings, multi-block messages with an odd XOF bit count, equal-length entry."""
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import KERNEL_PAIR
    eng = Engine(kernel=KERNEL_PAIR)
    algorithm, out_bits, vectors = load_kat_file(path)
    bits = xof_bits_for(algorithm, out_bits)
    msgs = [m for m, _ in vectors]
    for align, lead in ((1, 3), (4, 0), (8, 0)):
        got = device_digests(eng, algorithm, msgs, bits, align, lead)
        for row, (_, md) in zip(got, vectors):
            assert row.tobytes() == md
    rate = oracle.rate_bytes(algorithm)
    bits = 17 * rate + 3 if algorithm >= 4 else 0
    rng = np.random.default_rng(algorithm)
    msgs = [rng.integers(0, 256, int(n), dtype=np.uint8).tobytes() for n in rng.integers(0, 9 * rate, 777)]
    got = device_digests(eng, algorithm, msgs, bits)
    assert [r.tobytes() for r in got] == [oracle.hash_one(algorithm, m, bits) for m in msgs]
    host = oracle.generate_workload(3001 * 500, 500, seed=2)
    want = oracle.hash_batch(algorithm, host, fixed_len=500, count=3001, xof_bits=bits, workers=8)
    assert (eng.hash_fixed(algorithm, torch.from_numpy(host).cuda(), 500, 3001, bits).cpu().numpy() == want).all()
