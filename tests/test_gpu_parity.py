"""Parity tests proper: the CUDA path, called through the C ABI, against the
CPU oracle and the committed golden vectors -- bit-exact (bytes in, bytes out;
there is no floating point on this path)."""
import hashlib

import numpy as np
import pytest

from batches import materialize, ref_batch_cases
from conftest import all_kat_files, load_kat_file, xof_bits_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["auto", "no_warp_kernel"])
def engine(request):
    """Small-batch tests run twice: under the product default (batches of at most 3072
    multi-block messages take the warp-per-state kernel) and with that kernel switched off,
    so that the one-message-per-thread kernels see the same vectors.  Full-size tests use
    `big_engine` (the default) once."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import FLAG_NO_WARP_KERNEL
    return Engine(flags=FLAG_NO_WARP_KERNEL if request.param == "no_warp_kernel" else 0)


def pack(messages, align=1, lead=0):
    """Packs messages into one buffer with every start at `lead` mod `align`."""
    lengths = np.array([len(m) for m in messages], dtype=np.uint64)
    offsets = np.zeros(len(messages), dtype=np.uint64)
    pos = lead
    chunks = [b"\xEE" * lead]
    for i, m in enumerate(messages):
        pad = (-(pos - lead)) % align
        chunks.append(b"\xEE" * pad)
        pos += pad
        offsets[i] = pos
        chunks.append(bytes(m))
        pos += len(m)
    data = np.frombuffer(b"".join(chunks) + b"\xEE", dtype=np.uint8).copy()
    return data, offsets, lengths


def to_device(*arrays):
    import torch
    out = []
    for a in arrays:
        t = torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda()
        out.append(t)
    return out


def device_digests(engine, algorithm, messages, bits=0, align=1, lead=0, **kw):
    import torch
    data, offsets, lengths = pack(messages, align, lead)
    d, o, l = to_device(data, offsets, lengths)
    out = engine.hash_batch(algorithm, d, o, l, xof_output_bits=bits, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def test_native_library_is_loaded(big_engine):
    engine = big_engine
    from paper_1902_05320_b200 import library_path
    maps = open("/proc/self/maps").read()
    assert str(library_path()) in maps


def test_permutation_kat(big_engine, inline_kats, oracle):
    """Keccak-f[1600](0) (test_keccak.cpp:456-466) and random states vs the oracle."""
    engine = big_engine
    import torch
    rng = np.random.default_rng(11)
    states = rng.integers(0, 2**63, (1000, 25), dtype=np.uint64)
    states[0] = 0
    t = torch.from_numpy(states.view(np.int64).copy()).cuda()
    engine.permute_states(t)
    got = t.cpu().numpy().view(np.uint64)
    assert got[0].tobytes().hex() == inline_kats["keccak_f1600_zero_state"]["state"]
    for i in range(0, 1000, 37):
        assert (got[i] == oracle.permute(states[i])).all()


@pytest.mark.parametrize("path", all_kat_files(), ids=lambda p: p.stem)
def test_reference_vectors_device_path(engine, path):
    """All 892 .rsp vectors, each file as ONE batch (every length 0..R+16 and
    the long messages side by side in a warp), packed at odd offsets."""
    algorithm, out_bits, vectors = load_kat_file(path)
    bits = xof_bits_for(algorithm, out_bits)
    msgs = [m for m, _ in vectors]
    for align, lead in ((1, 0), (8, 0), (1, 3)):
        got = device_digests(engine, algorithm, msgs, bits, align, lead)
        for row, (_, md) in zip(got, vectors):
            assert row.tobytes() == md


@pytest.mark.parametrize("path", all_kat_files(), ids=lambda p: p.stem)
def test_reference_vectors_host_path(engine, path):
    """Same vectors through the host-buffer entry (the hash_batch drop-in)."""
    algorithm, out_bits, vectors = load_kat_file(path)
    got = engine.hash_messages(algorithm, [m for m, _ in vectors], xof_bits_for(algorithm, out_bits))
    assert got == [md for _, md in vectors]


def test_inline_kats(engine, inline_kats):
    for key, msg in (("empty_message", b""), ("msg_1600_bits_a3", b"\xa3" * 200)):
        for algorithm in range(6):
            bits = inline_kats[key]["xof_bits"][algorithm]
            got = engine.hash_messages(algorithm, [msg], bits)[0]
            assert got.hex() == inline_kats[key]["digests"][algorithm]
    assert engine.hash_messages("sha3_256", [b"abc"])[0].hex() == inline_kats["sha3_256_abc"]["digest"]


def test_hundred_copies_of_one_message(engine, oracle):
    """test_batch.cpp:102-111 (the paper's 10-byte example)."""
    msgs = [bytes([0x42] * 10)] * 100
    got = engine.hash_messages("sha3_256", msgs)
    assert got == [oracle.hash_one(1, msgs[0])] * 100


def test_variable_lengths_example(engine, oracle):
    """test_batch.cpp:169-176."""
    msgs = [b"", bytes([1] * 1000), bytes([5]), bytes([2] * 137)]
    assert engine.hash_messages("sha3_256", msgs) == [oracle.hash_one(1, m) for m in msgs]


def test_xof_328_bits_example(engine, oracle):
    """test_batch.cpp:150-160."""
    msgs = [bytes([1, 2, 3]), b"", bytes([9, 9, 9, 9])]
    got = engine.hash_messages("shake128", msgs, 328)
    assert [len(g) for g in got] == [41, 41, 41]
    assert got == [oracle.hash_one(4, m, 328) for m in msgs]


@pytest.mark.parametrize("case", ref_batch_cases(), ids=lambda c: c["name"])
def test_reference_batch_fixtures(engine, oracle, case):
    """Outputs of the compiled reference (tests/golden/ref_batches.json):
    multi-block squeeze, odd XOF bit counts, long and ragged batches -- device
    path (bucketed and not) and host path."""
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import FLAG_NO_BUCKETING
    msgs, _ = materialize(oracle, case["kind"], case["seed"], case["count"], case["max_len"])
    a, bits = case["algorithm"], case["xof_bits"]
    for got in (device_digests(engine, a, msgs, bits),
                device_digests(Engine(flags=FLAG_NO_BUCKETING), a, msgs, bits, align=8),
                np.stack([np.frombuffer(d, np.uint8) for d in engine.hash_messages(a, msgs, bits)])):
        assert got.shape == (case["count"], case["digest_bytes"])
        assert got[0].tobytes().hex() == case["first"]
        assert got[-1].tobytes().hex() == case["last"]
        assert hashlib.sha3_256(got.tobytes()).hexdigest() == case["checksum_sha3_256"]


@pytest.mark.parametrize("algorithm", range(6))
def test_block_boundary_lengths_vs_oracle(engine, oracle, algorithm):
    """Every length around the block boundaries (R-1: 0x06|0x80 in one byte; R:
    pad-only extra block), several alignments, several output lengths."""
    rate = oracle.rate_bytes(algorithm)
    rng = np.random.default_rng(100 + algorithm)
    lens = sorted(set(list(range(0, 20)) + list(range(rate - 10, rate + 10)) +
                      list(range(2 * rate - 3, 2 * rate + 3)) + [3 * rate, 7 * rate - 1, 5000]))
    msgs = [rng.integers(0, 256, n, dtype=np.uint8).tobytes() for n in lens]
    for bits in ([0] if algorithm < 4 else [8, 12, 8 * rate, 8 * rate + 8, 3 * 8 * rate + 5]):
        expect = [oracle.hash_one(algorithm, m, bits) for m in msgs]
        for align, lead in ((1, 0), (1, 5), (4, 0), (8, 0), (16, 0)):
            got = device_digests(engine, algorithm, msgs, bits, align, lead)
            assert [g.tobytes() for g in got] == expect, (bits, align, lead)


@pytest.mark.parametrize("algorithm,msg_len", [(0, 32), (0, 64), (0, 1024), (1, 64), (1, 136), (1, 200),
                                               (2, 32), (2, 128), (2, 512), (3, 72), (3, 1024), (3, 7),
                                               (4, 64), (5, 64), (1, 10), (1, 0)])
def test_fixed_length_batches(engine, oracle, algorithm, msg_len):
    """cfg2/cfg3-shaped batches at oracle-friendly sizes, device and host entries,
    on the reference's own synthetic stream."""
    import torch
    count = 3000
    total = max(count * msg_len, 1)
    bits = 0 if algorithm < 4 else 1024
    if msg_len:
        host = oracle.generate_workload(total, msg_len, seed=1)
        dev = engine.generate_workload(total, msg_len, seed=1)
        assert (dev.cpu().numpy() == host).all()      # device generator == workload.cpp
    else:
        host = np.zeros(1, np.uint8)
        dev = torch.zeros(16, dtype=torch.uint8, device="cuda")
    expect = oracle.hash_batch(algorithm, host, fixed_len=msg_len, count=count, xof_bits=bits, workers=4)
    got = engine.hash_fixed(algorithm, dev, msg_len, count, bits)
    torch.cuda.synchronize()
    assert (got.cpu().numpy() == expect).all()
    assert (engine.hash_fixed(algorithm, host, msg_len, count, bits) == expect).all()


def test_every_kernel_variant_agrees(big_engine, oracle):
    """The tuning matrix (unroll x FMA-offload presets, one-block and generic)
    must be invisible in the digests."""
    engine = big_engine
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import KERNEL_GENERIC, KERNEL_ONEBLOCK
    count = 5000
    host = oracle.generate_workload(count * 64, 64, seed=9)
    dev = torch.from_numpy(host).cuda()
    expect = oracle.hash_batch(1, host, fixed_len=64, count=count, workers=4)
    for unroll in (2, 4, 11, 20, 21, 22, 23, 24):
        for preset in range(9):
            e = Engine(kernel=KERNEL_ONEBLOCK, unroll=unroll, fma_preset=preset)
            got = e.hash_fixed("sha3_256", dev, 64, count)
            assert (got.cpu().numpy() == expect).all(), (unroll, preset)
    for preset in (0, 5):
        for threads in (64, 128, 256):
            e = Engine(kernel=KERNEL_GENERIC, fma_preset=preset, block_threads=threads)
            assert (e.hash_fixed("sha3_256", dev, 64, count).cpu().numpy() == expect).all()
    # SHAKE256 shares rate 17 / 32-byte output with SHA3-256 but not the pad byte
    expect_xof = oracle.hash_batch(5, host, fixed_len=64, count=count, xof_bits=256, workers=4)
    got = Engine(kernel=KERNEL_ONEBLOCK).hash_fixed("shake256", dev, 64, count, 256)
    assert (got.cpu().numpy() == expect_xof).all()


@pytest.mark.parametrize("algorithm,msg_len,bits", [
    (0, 32, 0), (0, 64, 0), (0, 128, 0), (1, 32, 0), (1, 64, 0), (1, 128, 0), (2, 32, 0), (2, 64, 0),
    (3, 32, 0), (3, 64, 0), (4, 32, 256), (4, 64, 256), (4, 128, 256), (4, 64, 512), (5, 64, 256),
    (5, 64, 512), (5, 32, 256), (5, 128, 256), (4, 64, 1024), (5, 64, 1024)])
def test_oneblock_shapes(oracle, algorithm, msg_len, bits):
    """Every instantiated shape of the single-block kernel, forced, vs the oracle; shapes
    without an instantiation must be refused (no silent substitution)."""
    import torch
    from paper_1902_05320_b200 import Engine, EngineError
    from paper_1902_05320_b200.engine import KERNEL_ONEBLOCK
    count = 4097
    host = oracle.generate_workload(count * msg_len, msg_len, seed=21)
    dev = torch.from_numpy(host).cuda()
    expect = oracle.hash_batch(algorithm, host, fixed_len=msg_len, count=count, xof_bits=bits, workers=4)
    got = Engine(kernel=KERNEL_ONEBLOCK).hash_fixed(algorithm, dev, msg_len, count, bits)
    assert (got.cpu().numpy() == expect).all()
    with pytest.raises(EngineError):
        Engine(kernel=KERNEL_ONEBLOCK).hash_fixed(algorithm, dev[:count * 24].contiguous(), 24, count, bits)


FEWBLOCK_SHAPES = ([(0, n, 0) for n in (256, 512, 1024)] + [(1, n, 0) for n in (256, 512, 1024)] +
                   [(2, n, 0) for n in (128, 256, 512, 1024)] + [(3, n, 0) for n in (128, 256, 512, 1024)] +
                   [(4, 64, 2048), (4, 64, 4096), (5, 64, 2048), (5, 64, 4096)])


@pytest.mark.parametrize("algorithm,msg_len,bits", FEWBLOCK_SHAPES)
def test_fewblock_shapes(oracle, algorithm, msg_len, bits):
    """Every instantiated shape of the static-shape multi-block kernel (kernel_fewblock.cu),
    forced, vs the oracle and vs the generic kernel; KERNEL_AUTO picks it for large batches of
    these shapes; shapes without an instantiation, odd-bit XOF lengths and misaligned buffers
    are refused when forced (and served by the generic kernel under AUTO)."""
    import torch
    from paper_1902_05320_b200 import Engine, EngineError, selected_kernel
    from paper_1902_05320_b200.engine import FLAG_NO_WARP_KERNEL, KERNEL_FEWBLOCK, KERNEL_GENERIC
    count = 4099
    host = oracle.generate_workload(count * msg_len, msg_len, seed=23)
    dev = torch.from_numpy(host).cuda()
    expect = oracle.hash_batch(algorithm, host, fixed_len=msg_len, count=count, xof_bits=bits, workers=4)
    forced = Engine(kernel=KERNEL_FEWBLOCK)
    got = forced.hash_fixed(algorithm, dev, msg_len, count, bits)
    assert (got.cpu().numpy() == expect).all()
    assert torch.equal(got, Engine(kernel=KERNEL_GENERIC).hash_fixed(algorithm, dev, msg_len, count, bits))
    assert selected_kernel(algorithm, msg_len, bits, 1 << 20).startswith("hash_fewblock_kernel<")
    auto = Engine(flags=FLAG_NO_WARP_KERNEL)
    assert torch.equal(got, auto.hash_fixed(algorithm, dev, msg_len, count, bits))
    # one message, and a count that leaves the last block of threads almost empty
    for n in (1, 129):
        assert (forced.hash_fixed(algorithm, dev, msg_len, n, bits).cpu().numpy() == expect[:n]).all()
    with pytest.raises(EngineError):  # not a whole number of lanes: neither the static nor the run-time-length form
        forced.hash_fixed(algorithm, dev[:count * (msg_len - 4)].contiguous(), msg_len - 4, count, bits)
    # a buffer that is only 8-byte aligned: refused when forced, the generic kernel under AUTO
    shifted = torch.empty(host.size + 8, dtype=torch.uint8, device="cuda")[8:]
    shifted.copy_(dev)
    with pytest.raises(EngineError):
        forced.hash_fixed(algorithm, shifted, msg_len, count, bits)
    assert (auto.hash_fixed(algorithm, shifted, msg_len, count, bits).cpu().numpy() == expect).all()
    if bits:  # an XOF length that rounds up to the same digest size but is not whole bytes
        with pytest.raises(EngineError):
            forced.hash_fixed(algorithm, dev, msg_len, count, bits - 3)
        odd = oracle.hash_batch(algorithm, host, fixed_len=msg_len, count=count, xof_bits=bits - 3, workers=4)
        assert (auto.hash_fixed(algorithm, dev, msg_len, count, bits - 3).cpu().numpy() == odd).all()


@pytest.mark.parametrize("algorithm,bits", [(0, 0), (1, 0), (2, 0), (3, 0), (4, 128), (4, 256), (4, 512),
                                            (5, 128), (5, 256), (5, 512)])
def test_manyblock_every_length(oracle, algorithm, bits):
    """The run-time-length form of the few-block kernel (hash_manyblock_kernel): equal-length
    messages of every whole number of lanes from the rate to just past three rate blocks -- every
    case of the final-block jump table with one, two and three whole blocks in front -- forced,
    vs the oracle; plus two long shapes, and the same batches under KERNEL_AUTO."""
    import torch
    from paper_1902_05320_b200 import Engine, EngineError, rate_bytes, selected_kernel
    from paper_1902_05320_b200.engine import FLAG_NO_WARP_KERNEL, KERNEL_FEWBLOCK
    rate = rate_bytes(algorithm)
    count = 131
    forced, auto = Engine(kernel=KERNEL_FEWBLOCK), Engine(flags=FLAG_NO_WARP_KERNEL)
    lengths = list(range(rate, 3 * rate + 17, 8)) + [5000 - 5000 % 8, 16 * rate]
    for msg_len in lengths:
        host = oracle.generate_workload(count * msg_len, msg_len, seed=29)
        dev = torch.from_numpy(host).cuda()
        expect = oracle.hash_batch(algorithm, host, fixed_len=msg_len, count=count, xof_bits=bits, workers=4)
        got = forced.hash_fixed(algorithm, dev, msg_len, count, bits)
        assert (got.cpu().numpy() == expect).all(), msg_len
        assert torch.equal(got, auto.hash_fixed(algorithm, dev, msg_len, count, bits)), msg_len
        name = selected_kernel(algorithm, msg_len, bits, 1 << 20)
        assert name.startswith("hash_manyblock_kernel<") or name.startswith("hash_fewblock_kernel<"), (msg_len, name)
    # below the rate, or not a whole number of lanes: not this kernel's
    for msg_len in (rate - 8, rate + 4):
        host = oracle.generate_workload(count * msg_len, msg_len, seed=29)
        with pytest.raises(EngineError):
            forced.hash_fixed(algorithm, torch.from_numpy(host).cuda(), msg_len, count, bits)


@pytest.mark.parametrize("algorithm", [4, 5])
@pytest.mark.parametrize("msg_len", [32, 64, 128])
@pytest.mark.parametrize("bits", [250, 255, 509, 1023])
def test_odd_bit_xof_on_oneblock_shapes(engine, oracle, algorithm, msg_len, bits):
    """XOF lengths that are not whole bytes but round up to a one-block digest size (32 / 64 /
    128 bytes): the last byte must come back masked (batch.cpp:22-24) through the device entry,
    the host entry, and the forced one-block / lane-split kernels must refuse the batch rather
    than return an unmasked byte."""
    import torch
    from paper_1902_05320_b200 import Engine, EngineError
    from paper_1902_05320_b200.engine import KERNEL_LANESPLIT, KERNEL_ONEBLOCK
    count = 1031
    host = oracle.generate_workload(count * msg_len, msg_len, seed=77)
    expect = oracle.hash_batch(algorithm, host, fixed_len=msg_len, count=count, xof_bits=bits)
    assert all(oracle.hash_one(algorithm, host[i * msg_len:(i + 1) * msg_len].tobytes(), bits)
               == expect[i].tobytes() for i in (0, 1, count - 1))
    mask = (1 << (bits % 8)) - 1
    assert (expect[:, -1] & ~np.uint8(mask) == 0).all() and (expect[:, -1] != 0).any()
    dev = torch.from_numpy(host).cuda()
    got = engine.hash_fixed(algorithm, dev, msg_len, count, bits)
    assert (got.cpu().numpy() == expect).all()
    assert (engine.hash_fixed(algorithm, host, msg_len, count, bits) == expect).all()
    for forced in (KERNEL_ONEBLOCK, KERNEL_LANESPLIT):
        with pytest.raises(EngineError):
            Engine(kernel=forced).hash_fixed(algorithm, dev, msg_len, count, bits)


@pytest.mark.parametrize("algorithm,msg_len,bits", [(1, 64, 0), (1, 8, 0), (1, 128, 0), (3, 64, 0),
                                                    (2, 96, 0), (5, 64, 512), (4, 160, 1344)])
def test_lanesplit_kernel(oracle, algorithm, msg_len, bits):
    """The lane-split comparison kernel (5 threads per state, shuffles + shared tile) gives
    the same digests; counts that do not fill the last warp / block included."""
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import KERNEL_LANESPLIT
    for count in (1, 5, 6, 7, 24, 25, 10_007):
        host = oracle.generate_workload(count * msg_len, msg_len, seed=31)
        dev = torch.from_numpy(np.concatenate([host, np.zeros(16, np.uint8)])).cuda()
        expect = oracle.hash_batch(algorithm, host, fixed_len=msg_len, count=count, xof_bits=bits)
        got = Engine(kernel=KERNEL_LANESPLIT).hash_fixed(algorithm, dev, msg_len, count, bits)
        assert (got.cpu().numpy() == expect).all(), count


@pytest.mark.parametrize("algorithm", range(6))
def test_staged_kernel(oracle, algorithm):
    """The TMA-staged comparison kernel (bulk async copies into shared memory, mbarrier
    completion): ragged batch with many multi-block messages at 8-byte aligned offsets, the
    same batch at odd offsets (nothing staged, direct path), and a fixed-length batch."""
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import KERNEL_STAGED
    rng = np.random.default_rng(70 + algorithm)
    rate = oracle.rate_bytes(algorithm)
    bits = 0 if algorithm < 4 else 8 * rate + 40
    lens = list(rng.integers(0, 12 * rate, 900)) + [rate + 15, rate + 16, rate + 17, 2 * rate + 16, 3 * rate,
                                                     5 * rate + 8, 40 * rate + 3]
    msgs = [rng.integers(0, 256, int(n), dtype=np.uint8).tobytes() for n in lens]
    expect = [oracle.hash_one(algorithm, m, bits) for m in msgs]
    eng = Engine(kernel=KERNEL_STAGED)
    for align, lead in ((8, 0), (16, 0), (8, 8), (1, 0), (8, 3)):
        got = device_digests(eng, algorithm, msgs, bits, align, lead)
        assert [g.tobytes() for g in got] == expect, (align, lead)
    count, msg_len = 3001, 4 * rate + 8
    host = oracle.generate_workload(count * msg_len, msg_len, seed=41)
    dev = torch.from_numpy(host).cuda()
    want = oracle.hash_batch(algorithm, host, fixed_len=msg_len, count=count, xof_bits=bits, workers=4)
    assert (eng.hash_fixed(algorithm, dev, msg_len, count, bits).cpu().numpy() == want).all()


def test_bucket_order_is_a_sorted_permutation(big_engine):
    """Device bucketing: every index exactly once; keys non-increasing, the key being the block
    count up to 128 blocks, 16 sub-bins per power of two above, and -- among single-block
    messages -- the number of whole 32-bit words (kernel_aux.cu: bucket_key)."""
    engine = big_engine
    import torch

    def key(lengths):
        blocks = lengths // 136 + 1
        e = np.floor(np.log2(np.maximum(blocks, 1))).astype(np.int64)
        coarse = 169 + (e - 7) * 16 + ((blocks >> np.maximum(e - 4, 0)) & 15)
        return np.where(blocks == 1, lengths >> 2, np.where(blocks <= 128, 40 + blocks, np.minimum(coarse, 511)))

    for lo, hi in ((1, 16384), (0, 135), (0, 400), (1, 200_000)):
        lengths = engine.generate_lengths(200_000, lo, hi, seed_len=2)
        order = engine.bucket_order("sha3_256", lengths).cpu().numpy().astype(np.int64)
        assert np.array_equal(np.sort(order), np.arange(200_000))
        host = lengths.cpu().numpy()
        keys = key(host)[order]
        assert (np.diff(keys) <= 0).all()
        blocks = (host // 136 + 1)[order]
        assert blocks[0] >= blocks.max() * 15 // 16 and blocks[-1] == blocks.min()
        if hi <= 16384:
            assert (np.diff(blocks) <= 0).all()      # up to 128 blocks every bin is one block count
    torch.cuda.synchronize()


def test_variable_length_workload_vs_oracle(engine, oracle):
    """cfg4-shaped batch (lengths 1..16 KiB from the device generator) on a
    subsample the oracle finishes quickly; bucketed == unbucketed == oracle."""
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import FLAG_NO_BUCKETING, splitmix64_at
    count = 4096
    lengths = engine.generate_lengths(count, 1, 16384, seed_len=2)
    host_len = lengths.cpu().numpy().astype(np.uint64)
    expect_len = 1 + splitmix64_at(np.uint64(2), np.arange(1, count + 1, dtype=np.uint64)) % np.uint64(16384)
    assert (host_len == expect_len).all()
    padded = (lengths + 7) // 8 * 8
    offsets = torch.cumsum(padded, 0) - padded
    data = torch.zeros(int(padded.sum().item()) + 16, dtype=torch.uint8, device="cuda")
    engine.fill_messages(data, offsets, lengths, seed=1)
    got = engine.hash_batch("sha3_256", data, offsets, lengths)
    got2 = Engine(flags=FLAG_NO_BUCKETING).hash_batch("sha3_256", data, offsets, lengths)
    torch.cuda.synchronize()
    expect = oracle.hash_batch(1, data.cpu().numpy(), offsets.cpu().numpy().astype(np.uint64), host_len,
                               workers=8)
    assert (got.cpu().numpy() == expect).all()
    assert (got2.cpu().numpy() == expect).all()
    # message content generator: word k of message i = splitmix(seed ^ i*C, k+1)
    i = 5
    key = np.uint64(1) ^ np.uint64((i * 0xd1342543de82ef95) & (2**64 - 1))
    n = int(host_len[i])
    words = splitmix64_at(key, np.arange(1, (n + 7) // 8 + 1, dtype=np.uint64)).view(np.uint8)[:n]
    off = int(offsets[i].item())
    assert (data[off:off + n].cpu().numpy() == words).all()


def test_full_size_properties_cfg1(big_engine, oracle):
    """cfg1 at full size (2^20 x 64 B): sampled digests vs the oracle, a checksum
    of all digests vs the oracle's, sharding invariance, and determinism."""
    engine = big_engine
    import torch
    count, total = 1 << 20, 1 << 26
    dev = engine.generate_workload(total, 64, seed=1)
    got = engine.hash_fixed("sha3_256", dev, 64, count)
    again = engine.hash_fixed("sha3_256", dev, 64, count)
    assert torch.equal(got, again)
    host = dev.cpu().numpy()
    expect = oracle.hash_batch(1, host, fixed_len=64, count=count, workers=8)
    g = got.cpu().numpy()
    assert hashlib.sha3_256(g.tobytes()).hexdigest() == hashlib.sha3_256(expect.tobytes()).hexdigest()
    # contiguous shards generated independently (as ranks do) give the same digests
    for first, n in ((0, 1000), (123_456, 4096), (count - 77, 77)):
        shard = engine.generate_workload(total, 64, seed=1, first_message=first, count=n)
        part = engine.hash_fixed("sha3_256", shard, 64, n)
        assert torch.equal(part, got[first:first + n])


def test_large_batch_roundtrip_properties(big_engine, oracle):
    """2^24 x 64 B (1 GiB): no oracle pass over everything -- sample 4096
    messages against the oracle and check the one-block and generic kernels agree
    on all 2^24 digests."""
    engine = big_engine
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import KERNEL_GENERIC
    count = 1 << 24
    dev = engine.generate_workload(count * 64, 64, seed=3)
    fast = engine.hash_fixed("sha3_256", dev, 64, count)
    slow = Engine(kernel=KERNEL_GENERIC).hash_fixed("sha3_256", dev, 64, count)
    assert torch.equal(fast, slow)
    idx = torch.randint(0, count, (4096,), generator=torch.Generator().manual_seed(5))
    msgs = dev.view(count, 64)[idx.cuda()].cpu().numpy()
    expect = oracle.hash_batch(1, msgs, fixed_len=64, count=4096, workers=8)
    assert (fast[idx.cuda()].cpu().numpy() == expect).all()


def test_host_entry_pipelined_equals_single_shot(big_engine, oracle):
    """Host-buffer entry with and without the chunked copy/compute pipeline
    (3 x 64 MiB slots), pageable and pinned memory."""
    engine = big_engine
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import FLAG_NO_PIPELINE
    count = 3_000_001               # ~183 MiB in: several chunks, ragged tail
    host = oracle.generate_workload(count * 64, 64, seed=4)
    a = engine.hash_fixed("sha3_256", host, 64, count)
    b = Engine(flags=FLAG_NO_PIPELINE).hash_fixed("sha3_256", host, 64, count)
    assert (a == b).all()
    pinned = torch.from_numpy(host).pin_memory()
    out = torch.empty((count, 32), dtype=torch.uint8).pin_memory()
    engine.hash_fixed_ptr("sha3_256", pinned.data_ptr(), 64, count, out.data_ptr())
    assert (out.numpy() == a).all()
    sample = np.arange(0, count, 9973)
    expect = oracle.hash_batch(1, host.reshape(count, 64)[sample], fixed_len=64, count=len(sample))
    assert (a[sample] == expect).all()


def test_reentrant_from_multiple_callers(big_engine, oracle):
    """test_batch.cpp:178-196: three threads, each with its own batch call."""
    engine = big_engine
    import threading
    rng = oracle.test_rng(54)
    msgs = [rng.random_bytes(rng.below(31)) for _ in range(200)]
    expect = [oracle.hash_one(1, m) for m in msgs]
    ok = [False] * 3

    def run(t):
        from paper_1902_05320_b200 import Engine
        ok[t] = Engine().hash_messages("sha3_256", msgs) == expect

    threads = [threading.Thread(target=run, args=(t,)) for t in range(3)]
    [t.start() for t in threads]
    [t.join() for t in threads]
    assert all(ok)


def test_xof_without_length_rejected_on_gpu_box_too(big_engine):
    engine = big_engine
    with pytest.raises(ValueError):
        engine.hash_messages("shake256", [b"\x01"], 0)


# ---- BASELINE.json configs at FULL size, through size-independent properties ----------

def _sample_check(oracle, algorithm, dev, msg_len, count, digests, bits=0, n=2048, seed=9):
    import torch
    idx = torch.randint(0, count, (n,), generator=torch.Generator().manual_seed(seed)).cuda()
    msgs = dev.view(count, msg_len)[idx].cpu().numpy()
    expect = oracle.hash_batch(algorithm, msgs, fixed_len=msg_len, count=n, xof_bits=bits, workers=8)
    assert (digests[idx].cpu().numpy() == expect).all()


def test_cfg5_full_size_2pow28(big_engine, oracle):
    """configs[4]: SHA3-256 over 2^28 x 64 B (16 GiB in, 8 GiB out).  Two independent kernels
    (single-block, fully unrolled vs generic, rolled) agree on every digest; 2048 sampled
    messages match the oracle; eight independently generated shards reproduce the digests
    (the N-GPU invariance); the first message is the cfg1/cfg5 stream KAT."""
    engine = big_engine
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import KERNEL_GENERIC
    count = 1 << 28
    dev = engine.generate_workload(count * 64, 64, seed=1)
    fast = engine.hash_fixed("sha3_256", dev, 64, count)
    slow = Engine(kernel=KERNEL_GENERIC).hash_fixed("sha3_256", dev, 64, count)
    assert torch.equal(fast, slow)
    del slow
    _sample_check(oracle, 1, dev, 64, count, fast)
    whole = int(fast.view(torch.int64).sum().item())
    parts = 0
    for rank in range(8):
        first, n = rank * (count // 8), count // 8
        shard = engine.generate_workload(count * 64, 64, seed=1, first_message=first, count=n)
        part = engine.hash_fixed("sha3_256", shard, 64, n)
        if rank in (0, 5):
            assert torch.equal(part, fast[first:first + n])
        parts = (parts + int(part.view(torch.int64).sum().item())) & (2**64 - 1)
        del shard, part
    assert parts == whole & (2**64 - 1)


@pytest.mark.parametrize("algorithm,msg_len,bits", [(0, 32, 0), (0, 1024, 0), (2, 256, 0), (3, 1024, 0),
                                                    (4, 64, 4096), (5, 64, 256), (5, 64, 2048)])
def test_cfg2_cfg3_full_size_2pow24(big_engine, oracle, algorithm, msg_len, bits):
    """configs[1] / configs[2] at 2^24 messages: auto-selected kernel == generic kernel on all
    digests, sampled oracle check, XOF prefix property (shorter output is a prefix)."""
    engine = big_engine
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import KERNEL_GENERIC
    count = 1 << 24
    dev = engine.generate_workload(count * msg_len, msg_len, seed=1)
    got = engine.hash_fixed(algorithm, dev, msg_len, count, bits)
    _sample_check(oracle, algorithm, dev, msg_len, count, got, bits, n=512)
    if msg_len <= 128:
        other = Engine(kernel=KERNEL_GENERIC).hash_fixed(algorithm, dev, msg_len, count, bits)
        assert torch.equal(got, other)
    if algorithm >= 4 and bits > 256:
        short = engine.hash_fixed(algorithm, dev, msg_len, count, 256)
        assert torch.equal(short, got[:, :32])          # test_sha3.cpp:150-158 at scale


def test_cfg4_full_size_2pow22(big_engine, oracle):
    """configs[3]: 2^22 messages, lengths 1..16 KiB (~34 GB): bucketed and unbucketed runs
    agree on every digest; 256 sampled messages match the oracle; digest slots follow input
    order although processing order is by block count."""
    engine = big_engine
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import FLAG_NO_BUCKETING
    count = 1 << 22
    lengths = engine.generate_lengths(count, 1, 16384, seed_len=2)
    padded = (lengths + 7) // 8 * 8
    offsets = torch.cumsum(padded, 0) - padded
    data = torch.empty(int(padded.sum().item()) + 16, dtype=torch.uint8, device="cuda")
    engine.fill_messages(data, offsets, lengths, seed=1)
    a = engine.hash_batch("sha3_256", data, offsets, lengths)
    b = Engine(flags=FLAG_NO_BUCKETING).hash_batch("sha3_256", data, offsets, lengths)
    assert torch.equal(a, b)
    idx = torch.randint(0, count, (256,), generator=torch.Generator().manual_seed(3))
    for i in idx.tolist():
        off, n = int(offsets[i].item()), int(lengths[i].item())
        assert a[i].cpu().numpy().tobytes() == oracle.hash_one(1, data[off:off + n].cpu().numpy().tobytes())


def test_one_huge_message_among_small_ones(engine):
    """Maximum-size edge: a 64 MiB message (493k blocks: the clamped top bucket) next to tiny
    ones, against hashlib (OpenSSL) -- the oracle's C loop would do too, hashlib is quicker."""
    import hashlib
    rng = np.random.default_rng(5)
    big = rng.integers(0, 256, 64 * 1024 * 1024 + 5, dtype=np.uint8).tobytes()
    msgs = [b"", big, b"abc", big[:136 * 300], bytes(200)]
    for alg, name in ((1, "sha3_256"), (3, "sha3_512")):
        assert engine.hash_messages(alg, msgs) == [hashlib.new(name, m).digest() for m in msgs]
    got = engine.hash_messages("shake128", msgs[1:3], 1344 * 2 + 8)
    assert got == [hashlib.shake_128(m).digest(337) for m in msgs[1:3]]


def test_variable_length_host_entry_pipelined(big_engine, oracle):
    """Host entry, packed ragged batch of ~200 MB: chunked 3-slot pipeline == single shot ==
    oracle (sampled); a batch whose offsets are NOT in order falls back to the single-shot
    path and is still right; permuting the messages permutes the digests."""
    engine = big_engine
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import FLAG_NO_PIPELINE
    rng = np.random.default_rng(12)
    count = 50_000
    lengths = rng.integers(0, 8192, count).astype(np.uint64)
    padded = (lengths + np.uint64(7)) // np.uint64(8) * np.uint64(8)
    offsets = (np.cumsum(padded) - padded).astype(np.uint64)
    data = rng.integers(0, 256, int(padded.sum()) + 16, dtype=np.uint8)
    piped = engine.hash_batch("sha3_384", data, offsets, lengths)
    single = Engine(flags=FLAG_NO_PIPELINE).hash_batch("sha3_384", data, offsets, lengths)
    assert (piped == single).all()
    sample = rng.choice(count, 300, replace=False)
    for i in sample:
        m = data[int(offsets[i]):int(offsets[i] + lengths[i])].tobytes()
        assert piped[i].tobytes() == oracle.hash_one(2, m)
    perm = rng.permutation(count)
    shuffled = engine.hash_batch("sha3_384", data, offsets[perm], lengths[perm])   # offsets out of order
    assert (shuffled == piped[perm]).all()


def test_pinned_alloc_api(big_engine):
    engine = big_engine
    import ctypes as C
    lib = engine.lib
    lib.b200sha3_pinned_alloc.argtypes = [C.c_uint64, C.POINTER(C.c_void_p)]
    lib.b200sha3_pinned_free.argtypes = [C.c_void_p]
    p = C.c_void_p()
    assert lib.b200sha3_pinned_alloc(1 << 20, C.byref(p)) == 0 and p.value
    buf = (C.c_uint8 * 64).from_address(p.value)
    for i in range(64):
        buf[i] = i
    out = np.zeros(32, dtype=np.uint8)
    engine.hash_fixed_ptr("sha3_256", p.value, 64, 1, out.ctypes.data)
    import hashlib
    assert out.tobytes() == hashlib.sha3_256(bytes(range(64))).digest()
    assert lib.b200sha3_pinned_free(p) == 0
    assert lib.b200sha3_pinned_alloc(0, C.byref(p)) == 0 and not p.value


def test_pageable_host_buffers_are_staged_through_the_bounce_ring(big_engine, oracle):
    """Host entries on ordinary (pageable) memory >= 4 MiB stage blocks through pinned bounce
    buffers with helper threads (csrc/capi_host.cu, BounceRing): every mix of pageable / pinned
    input and output, and a ragged batch whose offset / length tables are large enough to be
    staged too, must give the digests of the device-buffer entry."""
    engine = big_engine
    import torch
    count = 700_001                     # 42.7 MiB in, 21.4 MiB out: several 8 MiB blocks, ragged tail
    dev = engine.generate_workload(count * 64, 64, seed=9, count=count)
    want = engine.hash_fixed("sha3_256", dev, 64, count).cpu().numpy()
    pageable_in = dev.cpu().numpy().copy()
    pinned_in = torch.from_numpy(pageable_in).pin_memory()
    for src in (pageable_in.ctypes.data, pinned_in.data_ptr()):
        pageable_out = np.zeros((count, 32), dtype=np.uint8)
        pinned_out = torch.zeros((count, 32), dtype=torch.uint8).pin_memory()
        engine.hash_fixed_ptr("sha3_256", src, 64, count, pageable_out.ctypes.data)
        engine.hash_fixed_ptr("sha3_256", src, 64, count, pinned_out.data_ptr())
        assert (pageable_out == want).all() and (pinned_out.numpy() == want).all()

    rng = np.random.default_rng(21)
    count = 400_000                     # 6.4 MB of offsets + lengths
    lengths = rng.integers(0, 200, count).astype(np.uint64)
    offsets = (np.cumsum(lengths) - lengths).astype(np.uint64)        # unaligned starts
    data = rng.integers(0, 256, int(lengths.sum()) + 16, dtype=np.uint8)
    host = engine.hash_batch("shake256", data, offsets, lengths, 264)
    on_device = engine.hash_batch("shake256", torch.from_numpy(data).cuda(), torch.from_numpy(offsets).cuda(),
                                  torch.from_numpy(lengths).cuda(), 264).cpu().numpy()
    assert (host == on_device).all()
    for i in rng.choice(count, 200, replace=False):
        m = data[int(offsets[i]):int(offsets[i] + lengths[i])].tobytes()
        assert host[i].tobytes() == oracle.hash_one(5, m, 264)


@pytest.mark.parametrize("algorithm,bits", [(0, 0), (1, 0), (2, 0), (3, 0), (4, 128), (4, 256), (4, 512),
                                            (5, 128), (5, 256), (5, 512), (4, 328), (5, 1600)])
def test_all_short_ragged_batches(engine, oracle, algorithm, bits):
    """Variable-length batches in which every message is shorter than the rate go to
    hash_short_kernel (csrc/kernel_short.cu) when the starts are 8-byte aligned -- a choice made
    on the device from the classification flags.  Every length 0..rate-1 several times over, both
    layouts (aligned: short kernel; packed back to back: generic kernel), digest slots at an odd
    address, XOF lengths with and without an instantiation, and the same batch with one
    whole-block message appended (generic kernel) must all match the oracle."""
    import torch
    rate = oracle.rate_bytes(algorithm)
    rng = np.random.default_rng(100 + algorithm)
    lengths = np.concatenate([np.arange(rate), rng.integers(0, rate, 3000)]).astype(np.uint64)
    rng.shuffle(lengths)
    for align, extra in ((8, None), (1, None), (8, rate), (8, 5 * rate + 3)):
        lens = lengths if extra is None else np.concatenate([lengths, [np.uint64(extra)]]).astype(np.uint64)
        padded = (lens + np.uint64(align - 1)) // np.uint64(align) * np.uint64(align)
        offsets = (np.cumsum(padded) - padded).astype(np.uint64)
        data = rng.integers(0, 256, int(padded.sum()) + 16, dtype=np.uint8)
        expect = oracle.hash_batch(algorithm, data, offsets, lens, xof_bits=bits, workers=8)
        nbytes = expect.shape[1]
        d_out = torch.zeros(len(lens) * nbytes + 3, dtype=torch.uint8, device="cuda")
        for shift in (0, 3):    # digest array 16-byte aligned, then at an odd address
            out = d_out[shift:shift + len(lens) * nbytes].view(len(lens), nbytes)
            got = engine.hash_batch(algorithm, torch.from_numpy(data).cuda(), torch.from_numpy(offsets).cuda(),
                                    torch.from_numpy(lens).cuda(), bits, out=out)
            assert (got.cpu().numpy() == expect).all(), (align, extra, shift)
        host = engine.hash_batch(algorithm, data, offsets, lens, bits)      # host entry, same batch
        assert (host == expect).all(), (align, extra, "host")


@pytest.mark.parametrize("algorithm,bits", [(0, 0), (1, 0), (2, 0), (3, 0), (4, 256), (5, 512), (5, 128), (4, 1000)])
def test_equal_length_single_block_batches_of_every_length(big_engine, oracle, algorithm, bits):
    """Equal-length batches of every length 0 .. rate-1 (the paper's 10-byte messages among them,
    PAPER.md:307): lengths that are not 32 / 64 / 128 bytes go to hash_short_fixed_kernel
    (csrc/kernel_short.cu) with its uniform jump-table tails -- whole-lane loads when every
    start is 8-byte aligned, 4-byte loads + PRMT otherwise.  Device entry at three base
    alignments and the host entry, against the oracle."""
    engine = big_engine
    import torch
    rate = oracle.rate_bytes(algorithm)
    rng = np.random.default_rng(200 + algorithm)
    count = 257
    for msg_len in range(rate):
        data = rng.integers(0, 256, count * msg_len + 24, dtype=np.uint8)
        for lead in (0, 1, 4) if msg_len % 5 == 0 else (0,):
            view = data[lead:lead + count * msg_len]
            expect = oracle.hash_batch(algorithm, view, fixed_len=msg_len, count=count, xof_bits=bits, workers=4)
            dev = torch.from_numpy(data).cuda()[lead:lead + max(count * msg_len, 1)]
            got = engine.hash_fixed(algorithm, dev, msg_len, count, bits).cpu().numpy()
            assert (got == expect).all(), (msg_len, lead)
        host = engine.hash_fixed(algorithm, data[:max(count * msg_len, 1)], msg_len, count, bits)
        assert (host == oracle.hash_batch(algorithm, data[:count * msg_len], fixed_len=msg_len, count=count,
                                          xof_bits=bits, workers=4)).all(), (msg_len, "host")


def test_empty_messages_do_not_widen_the_host_range(big_engine, oracle):
    """An empty message's offset means nothing: it must not extend the byte range the host
    entry copies (offsets far outside the buffer, NULL data with all-empty batches)."""
    import ctypes as C
    engine = big_engine
    data = np.frombuffer(b"0123456789", dtype=np.uint8).copy()
    offsets = np.array([0, 1 << 40, 3, (1 << 63) + 5], dtype=np.uint64)
    lengths = np.array([10, 0, 4, 0], dtype=np.uint64)
    got = engine.hash_batch("sha3_256", data, offsets, lengths)
    expect = [oracle.hash_one(1, m) for m in (b"0123456789", b"", b"3456", b"")]
    assert [g.tobytes() for g in got] == expect
    # the same shape inside a long in-order batch (the strip fast path must notice the empty one)
    n = 5000
    lengths = np.full(n, 7, dtype=np.uint64)
    offsets = np.arange(n, dtype=np.uint64) * np.uint64(7)
    lengths[1234] = 0
    offsets[1234] = np.uint64(1 << 50)
    blob = np.random.default_rng(1).integers(0, 256, 7 * n, dtype=np.uint8)
    got = engine.hash_batch("sha3_224", blob, offsets, lengths)
    for i in (0, 1233, 1234, 1235, n - 1):
        m = blob[int(offsets[i]):int(offsets[i]) + int(lengths[i])].tobytes() if lengths[i] else b""
        assert got[i].tobytes() == oracle.hash_one(0, m)
    # all-empty batch with NULL data and arbitrary offsets
    out = np.zeros((3, 32), dtype=np.uint8)
    offs = np.array([5, 1 << 44, 77], dtype=np.uint64)
    lens = np.zeros(3, dtype=np.uint64)
    rc = engine.lib.b200sha3_hash_batch(1, None, offs.ctypes.data, lens.ctypes.data, 3, 0, out.ctypes.data, None)
    assert rc == 0 and all(out[i].tobytes() == oracle.hash_one(1, b"") for i in range(3))


def test_long_messages_are_cut_into_chunks_by_bytes(big_engine):
    """Fewer than 1024 messages but more than the 1 GiB chunk target: the host entry must
    close chunks by BYTES (copy / compute overlap, bounded device staging), digests unchanged."""
    import hashlib
    engine = big_engine
    rng = np.random.default_rng(12)
    n = 700
    lengths = rng.integers(2_000_000, 2_400_000, n).astype(np.uint64)          # ~1.5 GB in all
    offsets = np.concatenate([[0], np.cumsum((lengths + 7) // 8 * 8)[:-1]]).astype(np.uint64)
    total = int(offsets[-1] + lengths[-1])
    blob = rng.integers(0, 2**63, total // 8 + 2, dtype=np.uint64).view(np.uint8)
    got = engine.hash_batch("sha3_256", blob, offsets, lengths)
    assert engine.last_kernel_launches >= 2                                    # more than one chunk
    for i in (0, 1, 299, 480, 698, 699):
        m = blob[int(offsets[i]):int(offsets[i] + lengths[i])].tobytes()
        assert got[i].tobytes() == hashlib.sha3_256(m).digest()
    import torch
    dev = engine.hash_batch("sha3_256", torch.from_numpy(blob).cuda(), torch.from_numpy(offsets.view(np.int64)).cuda(),
                            torch.from_numpy(lengths.view(np.int64)).cuda())
    assert (dev.cpu().numpy() == got).all()


def test_device_entries_can_be_captured_in_a_cuda_graph(oracle):
    """The device-buffer entries only enqueue work (kernels, stream-ordered scratch, an event
    fork / join for the two alternative kernels of a variable-length batch), so a caller can
    capture them in a CUDA graph and replay it on new data in the same buffers."""
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import FLAG_NO_WARP_KERNEL
    eng = Engine(flags=FLAG_NO_WARP_KERNEL)      # the multi-launch path: bucketing + both hash kernels
    rng = np.random.default_rng(5)
    count = 3000
    lengths = rng.integers(0, 130, count).astype(np.uint64)
    offsets = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.uint64)
    blob = rng.integers(0, 256, int(lengths.sum()) + 16, dtype=np.uint8)
    d, o, l = to_device(blob, offsets, lengths)
    fixed = torch.from_numpy(rng.integers(0, 256, 4096 * 64, dtype=np.uint8)).cuda()
    out_var = torch.empty((count, 32), dtype=torch.uint8, device="cuda")
    out_fix = torch.empty((4096, 32), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):              # warm-up outside the capture (pools, side lane)
        eng.hash_batch("sha3_256", d, o, l, out=out_var)
        eng.hash_fixed("sha3_256", fixed, 64, 4096, out=out_fix)
    torch.cuda.current_stream().wait_stream(stream)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        eng.hash_batch("sha3_256", d, o, l, out=out_var)
        eng.hash_fixed("sha3_256", fixed, 64, 4096, out=out_fix)
    for trial in range(3):                       # new bytes in the same buffers, replay
        blob2 = rng.integers(0, 256, blob.size, dtype=np.uint8)
        fixed2 = rng.integers(0, 256, 4096 * 64, dtype=np.uint8)
        d.copy_(torch.from_numpy(blob2))
        fixed.copy_(torch.from_numpy(fixed2))
        out_var.zero_()
        out_fix.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert (out_var.cpu().numpy() == oracle.hash_batch(1, blob2, offsets, lengths, workers=4)).all()
        assert (out_fix.cpu().numpy() == oracle.hash_batch(1, fixed2, fixed_len=64, count=4096, workers=4)).all()


@pytest.mark.parametrize("algorithm,bits", [(1, 0), (3, 0), (4, 1027)])
def test_few_long_messages_from_pinned_memory_are_hashed_in_pieces(big_engine, algorithm, bits):
    """Few long equal-length messages in pinned host memory take the piece pipeline of the
    fixed-length host entry (strided copies of one piece of every message, absorbed by the
    incremental warp kernel while the next piece is on the link): same digests as hashlib, as
    the unpipelined call and as the device entry; lengths that are no multiple of the rate or
    of the piece size."""
    import hashlib
    import torch
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import FLAG_NO_PIPELINE
    engine = big_engine
    names = ["sha3_224", "sha3_256", "sha3_384", "sha3_512", "shake_128", "shake_256"]
    for count, msg_len in ((96, 1_000_003), (700, 300_001)):
        host = torch.randint(0, 256, (count * msg_len,), dtype=torch.uint8).pin_memory()
        nbytes = (bits + 7) // 8 if algorithm >= 4 else (28, 32, 48, 64)[algorithm]
        out = torch.zeros(count * nbytes, dtype=torch.uint8).pin_memory()
        engine.hash_fixed_ptr(algorithm, host.data_ptr(), msg_len, count, out.data_ptr(), bits)
        assert engine.last_kernel_launches > 3                  # one update per piece + the finish
        got = out.view(count, nbytes).numpy()
        plain = Engine(flags=FLAG_NO_PIPELINE).hash_fixed(algorithm, host.numpy(), msg_len, count, bits)
        assert (got == plain).all()
        dev = engine.hash_fixed(algorithm, host.cuda(), msg_len, count, bits).cpu().numpy()
        assert (got == dev).all()
        raw = host.numpy()
        for i in (0, 1, count // 2, count - 1):
            h = hashlib.new(names[algorithm], raw[i * msg_len:(i + 1) * msg_len].tobytes())
            want = h.digest(nbytes) if algorithm >= 4 else h.digest()
            if algorithm >= 4 and bits % 8:
                want = want[:-1] + bytes([want[-1] & ((1 << (bits % 8)) - 1)])
            assert got[i].tobytes() == want
