"""Batched incremental hashing on the device: the reference's
SpongeHasher / Hasher properties (proj/tests/test_sponge.cpp:114-194,
proj/tests/test_sha3.cpp:205-246) restated for N streams at once."""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HASHLIB = ["sha3_224", "sha3_256", "sha3_384", "sha3_512", "shake_128", "shake_256"]


@pytest.fixture(scope="module", params=["auto", "no_warp_kernel"])
def engine(request):
    """Every test runs on both forms of the incremental kernels: one stream per warp (what
    KERNEL_AUTO picks for the few hundred streams used here) and one stream per thread."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1902_05320_b200 import Engine
    from paper_1902_05320_b200.engine import FLAG_NO_WARP_KERNEL
    return Engine(flags=FLAG_NO_WARP_KERNEL if request.param == "no_warp_kernel" else 0)


def feed(hasher, messages, cuts, rng):
    """Feeds message i in pieces ending at cuts[i][k]; round k sends piece k of every stream
    (zero-length where a stream has fewer pieces), packed at random byte offsets."""
    import torch
    rounds = max(len(c) for c in cuts)
    for k in range(rounds):
        pieces = [m[(c[k - 1] if k else 0):c[k]] if k < len(c) else b"" for m, c in zip(messages, cuts)]
        lengths = np.array([len(p) for p in pieces], dtype=np.int64)
        gaps = rng.integers(0, 4, len(pieces))
        offsets = np.zeros(len(pieces), dtype=np.int64)
        blob, pos = [], 0
        for i, p in enumerate(pieces):
            blob.append(b"\xEE" * int(gaps[i]))
            pos += int(gaps[i])
            offsets[i] = pos
            blob.append(p)
            pos += len(p)
        data = np.frombuffer(b"".join(blob) + b"\xEE" * 8, dtype=np.uint8).copy()
        hasher.update(torch.from_numpy(data).cuda(), torch.from_numpy(offsets).cuda(),
                      torch.from_numpy(lengths).cuda())


@pytest.mark.parametrize("algorithm", range(6))
def test_chunked_update_equals_one_shot(engine, oracle, algorithm):
    """test_sponge.cpp:114-132 at batch scale: any chunking of the input gives the one-shot
    digest -- chunk boundaries at every position relative to the block, empty chunks, streams
    of different lengths."""
    from paper_1902_05320_b200 import BatchHasher
    rng = np.random.default_rng(40 + algorithm)
    rate = oracle.rate_bytes(algorithm)
    n = 600
    messages = [rng.integers(0, 256, int(L), dtype=np.uint8).tobytes()
                for L in rng.integers(0, 4 * rate + 50, n)]
    messages[:4] = [b"", bytes(rate), bytes(rate - 1), bytes(2 * rate)]
    cuts = []
    for m in messages:
        k = int(rng.integers(1, 6))
        c = sorted(int(x) for x in rng.integers(0, len(m) + 1, k - 1)) + [len(m)]
        cuts.append(c)
    h = BatchHasher(algorithm, n, engine)
    feed(h, messages, cuts, rng)
    bits = 0 if algorithm < 4 else 8 * rate + 24          # XOF: more than one squeeze block
    got = (h.digest() if algorithm < 4 else h.finish(bits)).cpu().numpy()
    for i, m in enumerate(messages):
        assert got[i].tobytes() == oracle.hash_one(algorithm, m, bits), (i, len(m), cuts[i])
    # reset() gives fresh states (Hasher::reset)
    h.reset()
    feed(h, messages, [[len(m)] for m in messages], rng)
    again = (h.digest() if algorithm < 4 else h.finish(bits)).cpu().numpy()
    assert (again == got).all()


@pytest.mark.parametrize("algorithm", [4, 5])
def test_chunked_squeeze_equals_one_shot(engine, oracle, algorithm):
    """test_sponge.cpp:134-150: reading 500 bytes in uneven pieces == one 500-byte read;
    finish(bits) followed by read() continues the same stream."""
    import torch
    from paper_1902_05320_b200 import BatchHasher
    rng = np.random.default_rng(50 + algorithm)
    n = 300
    messages = [rng.integers(0, 256, int(L), dtype=np.uint8).tobytes() for L in rng.integers(0, 400, n)]
    expect = [oracle.hash_one(algorithm, m, 8 * 500) for m in messages]
    h = BatchHasher(algorithm, n, engine)
    feed(h, messages, [[len(m)] for m in messages], rng)
    assert h.finish(0) is None
    parts = [h.read(k) for k in (1, 7, 160, 8, 168, 136, 20)]
    out = torch.cat(parts, dim=1).cpu().numpy()
    assert out.shape == (n, 500)
    assert [out[i].tobytes() for i in range(n)] == expect
    h.reset()
    feed(h, messages, [[len(m)] for m in messages], rng)
    first = h.finish(8 * 100).cpu().numpy()
    rest = h.read(400).cpu().numpy()
    assert [first[i].tobytes() + rest[i].tobytes() for i in range(n)] == expect


def test_state_machine_misuse(engine):
    """test_sponge.cpp:173-194 / Hasher misuse (sha3.cpp:103-126): logic errors, not wrong output."""
    import torch
    from paper_1902_05320_b200 import BatchHasher, EngineStateError
    data = torch.zeros(64, dtype=torch.uint8, device="cuda")
    h = BatchHasher("sha3_256", 4, engine)
    h.update(data, chunk_len=16)
    with pytest.raises(EngineStateError):
        h.finish()                      # finish()/read() is for XOFs
    with pytest.raises(EngineStateError):
        h.read(8)                       # squeeze before finish
    h.digest()
    with pytest.raises(EngineStateError):
        h.update(data, chunk_len=16)    # update after finish
    with pytest.raises(EngineStateError):
        h.digest()                      # finish twice
    x = BatchHasher("shake128", 4, engine)
    with pytest.raises(EngineStateError):
        x.digest()                      # digest() is for hash variants
    with pytest.raises(EngineStateError):
        x.read(8)
    x.finish(0)
    x.read(8)
    with pytest.raises(EngineStateError):
        x.update(data, chunk_len=16)
    with pytest.raises(ValueError):
        BatchHasher(9, 4, engine)


def test_one_long_stream_in_pieces(engine):
    """A single 48 MiB input that never sits in one buffer: 1 MiB pieces (odd sizes) against
    hashlib -- what the streaming front end is for."""
    import torch
    from paper_1902_05320_b200 import BatchHasher
    rng = np.random.default_rng(60)
    total = 48 * 1024 * 1024 + 13
    blob = rng.integers(0, 256, total, dtype=np.uint8)
    ref = hashlib.sha3_256()
    h = BatchHasher("sha3_256", 1, engine)
    pos = 0
    while pos < total:
        n = min(total - pos, int(rng.integers(900_000, 1_200_000)))
        piece = blob[pos:pos + n]
        ref.update(piece.tobytes())
        h.update(torch.from_numpy(piece.copy()).cuda(), chunk_len=n)
        pos += n
    assert h.digest().cpu().numpy()[0].tobytes() == ref.digest()


@pytest.mark.parametrize("algorithm", [1, 3, 4])
def test_warp_and_thread_forms_share_the_states(oracle, algorithm):
    """The two forms of the incremental kernels keep the same state layout in HBM: updates may
    alternate between them on one set of states, and either may finish / squeeze."""
    import torch
    from paper_1902_05320_b200 import BatchHasher, Engine
    from paper_1902_05320_b200.engine import FLAG_NO_WARP_KERNEL
    rng = np.random.default_rng(90 + algorithm)
    rate = oracle.rate_bytes(algorithm)
    n = 300
    engines = [Engine(), Engine(flags=FLAG_NO_WARP_KERNEL)]
    messages = [rng.integers(0, 256, int(L), dtype=np.uint8).tobytes() for L in rng.integers(0, 6 * rate, n)]
    h = BatchHasher(algorithm, n, engines[0])
    done = [0] * n
    for step in range(5):                       # five rounds of pieces, alternating the form
        h.engine = engines[step % 2]
        take = [int(rng.integers(0, len(m) - d + 1)) if step < 4 else len(m) - d for m, d in zip(messages, done)]
        lengths = np.array(take, dtype=np.int64)
        offsets = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
        blob = b"".join(m[d:d + k] for m, d, k in zip(messages, done, take)) + b"\0" * 8
        h.update(torch.from_numpy(np.frombuffer(blob, dtype=np.uint8).copy()).cuda(),
                 torch.from_numpy(offsets).cuda(), torch.from_numpy(lengths).cuda())
        done = [d + k for d, k in zip(done, take)]
    if algorithm < 4:
        got = h.digest().cpu().numpy()
        want = [oracle.hash_one(algorithm, m) for m in messages]
    else:
        h.engine = engines[1]
        first = h.finish(8 * 100).cpu().numpy()                      # 100 bytes by the thread form ...
        h.engine = engines[0]
        more = h.read(2 * rate + 7).cpu().numpy()                    # ... the rest by the warp form
        got = np.concatenate([first, more], axis=1)
        want = [oracle.hash_one(algorithm, m, 8 * (100 + 2 * rate + 7)) for m in messages]
    assert [g.tobytes() for g in got] == want
    h.close()
