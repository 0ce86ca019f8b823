"""Pins the CPU oracle (oracle/keccak_oracle.c) before anything trusts it:
against the reference's 892 on-disk vectors, its inline KATs, hashlib, and --
where oracle/_ref exists -- the compiled reference itself."""
import hashlib
import re

import numpy as np
import pytest

from conftest import GOLDEN, REFERENCE_ROOT, all_kat_files, load_kat_file, reference_style_batch, xof_bits_for

HASHLIB = ["sha3_224", "sha3_256", "sha3_384", "sha3_512", "shake_128", "shake_256"]


def hashlib_digest(algorithm, msg, xof_bits=0):
    h = hashlib.new(HASHLIB[algorithm], msg)
    if algorithm >= 4:
        out = bytearray(h.digest((xof_bits + 7) // 8))
        if xof_bits % 8:
            out[-1] &= (1 << (xof_bits % 8)) - 1
        return bytes(out)
    return h.digest()


def test_golden_inventory():
    files = all_kat_files()
    assert len(files) == 12
    assert sum(len(load_kat_file(f)[2]) for f in files) == 892


@pytest.mark.parametrize("path", all_kat_files(), ids=lambda p: p.stem)
def test_oracle_matches_reference_vectors(oracle, path):
    algorithm, out_bits, vectors = load_kat_file(path)
    for msg, md in vectors:
        assert oracle.hash_one(algorithm, msg, xof_bits_for(algorithm, out_bits)) == md


@pytest.mark.parametrize("path", all_kat_files(), ids=lambda p: p.stem)
def test_oracle_batch_entry_matches_reference_vectors(oracle, path):
    """Same vectors through the packed-buffer batch entry, 3 workers."""
    from oracle.binding import pack
    algorithm, out_bits, vectors = load_kat_file(path)
    data, offsets, lengths = pack([m for m, _ in vectors])
    got = oracle.hash_batch(algorithm, data, offsets, lengths,
                            xof_bits=xof_bits_for(algorithm, out_bits), workers=3)
    for row, (_, md) in zip(got, vectors):
        assert row.tobytes() == md


def test_inline_kats(oracle, inline_kats):
    for key, msg in (("empty_message", b""), ("msg_1600_bits_a3", b"\xa3" * 200)):
        for algorithm in range(6):
            bits = inline_kats[key]["xof_bits"][algorithm]
            assert oracle.hash_one(algorithm, msg, bits).hex() == inline_kats[key]["digests"][algorithm]
    assert oracle.hash_one(1, b"abc").hex() == inline_kats["sha3_256_abc"]["digest"]


def test_permutation_kat(oracle, inline_kats):
    out = oracle.permute(np.zeros(25, dtype=np.uint64))
    assert out.tobytes().hex() == inline_kats["keccak_f1600_zero_state"]["state"]


def test_inline_kats_match_reference_sources(inline_kats):
    """The typed-in constants are the reference's (only checkable where it is mounted)."""
    tests = REFERENCE_ROOT / "proj" / "tests"
    if not tests.exists():
        pytest.skip("reference not mounted")
    text = "".join((tests / f).read_text() for f in ("acceptance.cpp", "test_keccak.cpp", "test_bench.cpp", "test_sha3.cpp"))
    flat = re.sub(r'"\s*\n\s*"', "", text)
    for key in ("empty_message", "msg_1600_bits_a3"):
        for d in inline_kats[key]["digests"]:
            assert d in flat
    assert inline_kats["sha3_256_abc"]["digest"] in flat
    assert inline_kats["keccak_f1600_zero_state"]["state"] in flat


def test_golden_files_are_the_reference_vectors():
    """tests/golden/*.kat carries exactly what proj/tests/vectors/*.rsp holds."""
    src = REFERENCE_ROOT / "proj" / "tests" / "vectors"
    if not src.exists():
        pytest.skip("reference not mounted")
    for kat in all_kat_files():
        _, _, vectors = load_kat_file(kat)
        rsp = (src / (kat.stem + ".rsp")).read_text()
        mds = re.findall(r"^MD = ([0-9a-f]+)$", rsp, flags=re.M)
        assert mds == [md.hex() for _, md in vectors]
        lens = [int(x) for x in re.findall(r"^Len = (\d+)$", rsp, flags=re.M)]
        assert lens == [8 * len(m) for m, _ in vectors]


def test_oracle_vs_hashlib_edge_lengths(oracle):
    """Block-boundary lengths and multi-block squeezes (the .rsp files stop at
    256 output bits)."""
    rng = np.random.default_rng(7)
    for algorithm in range(6):
        rate = oracle.rate_bytes(algorithm)
        for n in (0, 1, 7, 8, 9, rate - 9, rate - 8, rate - 2, rate - 1, rate, rate + 1, 2 * rate - 1,
                  2 * rate, 2 * rate + 1, 5 * rate + 3, 4096):
            msg = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
            for bits in ([0] if algorithm < 4 else [1, 7, 8, 12, 328, 8 * rate - 8, 8 * rate, 8 * rate + 8,
                                                    8 * rate + 3, 4096, 4099, 16 * rate + 8]):
                assert oracle.hash_one(algorithm, msg, bits) == hashlib_digest(algorithm, msg, bits)


def test_xof_prefix_and_bit_mask(oracle):
    """proj/tests/test_sha3.cpp:150-168."""
    rng = oracle.test_rng(43)
    msg = rng.random_bytes(100)
    for a in (4, 5):
        small, big = oracle.hash_one(a, msg, 128), oracle.hash_one(a, msg, 4096)
        assert big[:len(small)] == small
    rng = oracle.test_rng(44)
    msg = rng.random_bytes(17)
    full, partial = oracle.hash_one(5, msg, 16), oracle.hash_one(5, msg, 12)
    assert len(partial) == 2 and partial[0] == full[0] and partial[1] == (full[1] & 0x0F)


def test_validation(oracle):
    with pytest.raises(ValueError):
        oracle.hash_one(5, b"\x01", 0)      # XOF without length: batch.cpp:66-68
    assert oracle.digest_bytes(1, 999) == 32  # hashes ignore xof_output_bits
    assert oracle.hash_one(1, b"abc", 999) == oracle.hash_one(1, b"abc")
    assert [oracle.rate_bytes(a) for a in range(6)] == [144, 136, 104, 72, 168, 136]


def test_workload_generator(oracle, inline_kats):
    """workload.cpp:16-47: first message of the cfg1 stream, and odd sizes."""
    w = oracle.generate_workload(1 << 26, 64, seed=1)
    assert len(w) == 1 << 26
    assert hashlib.sha3_256(w[:64].tobytes()).hexdigest() == \
        inline_kats["workload_cfg1_first_message_sha3_256"]["digest"]
    from paper_1902_05320_b200.engine import splitmix64_at
    first = splitmix64_at(np.uint64(1), np.arange(1, 9, dtype=np.uint64)).view(np.uint8).tobytes()
    assert hashlib.sha3_256(first).hexdigest() == \
        inline_kats["splitmix64_seed1_first_64_bytes_sha3_256"]["digest"]
    w10 = oracle.generate_workload(1202, 10, seed=1)   # the paper's 10-byte messages
    assert len(w10) == 1200
    seed = np.uint64((1 ^ (1202 * 0x9e3779b97f4a7c15)) & (2**64 - 1))
    words = splitmix64_at(seed, np.arange(1, 241, dtype=np.uint64))
    expect = np.concatenate([np.concatenate([words[2 * i:2 * i + 1].view(np.uint8),
                                             words[2 * i + 1:2 * i + 2].view(np.uint8)[:2]])
                             for i in range(120)])
    assert (w10 == expect).all()


# ---- against the compiled reference (oracle/_ref) -------------------------

def test_reference_agrees_on_vectors(reference):
    for path in all_kat_files():
        algorithm, out_bits, vectors = load_kat_file(path)
        for msg, md in vectors[::7]:
            assert reference.one_shot(algorithm, msg, xof_bits_for(algorithm, out_bits)) == md


def test_reference_permutation(reference, oracle):
    rng = np.random.default_rng(3)
    for _ in range(50):
        s = rng.integers(0, 2**63, 25, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, 25, dtype=np.uint64)
        assert (reference.permute(s) == oracle.permute(s)).all()


@pytest.mark.parametrize("seed,counts,max_len", [(52, (0, 1, 7, 100, 2000), 300),
                                                 (0xE9, (0, 1, 7, 100, 10000), 199)])
def test_oracle_equals_reference_hash_batch(reference, oracle, seed, counts, max_len):
    """The batches of test_batch.cpp:119-135 and acceptance.cpp:254-273, reference
    (sequential and parallel) vs oracle, all six variants."""
    from oracle.binding import pack
    rng = oracle.test_rng(seed)
    for count in counts:
        msgs = [rng.random_bytes(rng.below(max_len + 1)) for _ in range(count)]
        data, offsets, lengths = pack(msgs)
        for algorithm in range(6):
            bits = (0, 0, 0, 0, 4099, 328)[algorithm]
            seq = reference.hash_batch(algorithm, data, offsets, lengths, xof_bits=bits, parallel=False)
            par = reference.hash_batch(algorithm, data, offsets, lengths, xof_bits=bits, parallel=True,
                                       workers=3, chunk=5)
            mine = oracle.hash_batch(algorithm, data, offsets, lengths, xof_bits=bits, workers=2)
            assert (seq == par).all() and (seq == mine).all()


def test_reference_rejects_xof_without_length(reference):
    with pytest.raises(ValueError):
        reference.hash_batch(5, np.zeros(1, np.uint8), np.zeros(1, np.uint64), np.ones(1, np.uint64))


def test_reference_workload_equals_oracle(reference, oracle):
    for total, size in ((1202, 10), (1 << 16, 64), (100003, 137), (4096, 8)):
        assert (reference.generate_workload(total, size) == oracle.generate_workload(total, size)).all()


def test_oracle_matches_reference_batch_fixtures(oracle):
    """tests/golden/ref_batches.json: outputs of the compiled reference for
    multi-block squeezes, odd XOF lengths, long and variable-length batches."""
    from batches import materialize, ref_batch_cases
    from oracle.binding import pack
    for case in ref_batch_cases():
        msgs, _ = materialize(oracle, case["kind"], case["seed"], case["count"], case["max_len"])
        data, offsets, lengths = pack(msgs)
        got = oracle.hash_batch(case["algorithm"], data, offsets, lengths, xof_bits=case["xof_bits"],
                                workers=4)
        assert got.shape[1] == case["digest_bytes"]
        assert got[0].tobytes().hex() == case["first"], case["name"]
        assert got[-1].tobytes().hex() == case["last"], case["name"]
        assert hashlib.sha3_256(got.tobytes()).hexdigest() == case["checksum_sha3_256"], case["name"]
