"""ctypes bindings of the two CPU checkers.  TEST INFRASTRUCTURE ONLY.

* ``Oracle``     -- oracle/liboracle.so, the C restatement (keccak_oracle.c).
* ``Reference``  -- oracle/_ref/libsha3kit_ref.so, the reference's own core
  library compiled from /root/reference by oracle/Makefile (present in the build
  container and shipped prebuilt to the GPU box; ``Reference.available()`` says
  whether it is there).

Both take packed buffers: ``data`` (uint8), optional ``offsets``/``lengths``
(uint64) or a fixed message length, and return a (count, digest_bytes) uint8
array in message order.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libsha3kit_ref.so"
REF_HASHINTO_SO = HERE / "_ref" / "libsha3kit_ref_hashinto.so"

ALGORITHMS = ("sha3_224", "sha3_256", "sha3_384", "sha3_512", "shake128", "shake256")
u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)


def build(quiet: bool = True) -> None:
    """(Re)builds liboracle.so and, when /root/reference is present, _ref."""
    subprocess.run(["make", "-C", str(HERE)], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _ptr(a, typ):
    if a is None:
        return C.cast(None, typ)
    return a.ctypes.data_as(typ)


def _as_u8(buf) -> np.ndarray:
    if isinstance(buf, np.ndarray):
        return np.ascontiguousarray(buf, dtype=np.uint8).reshape(-1)
    return np.frombuffer(bytes(buf), dtype=np.uint8)


def pack(messages):
    """list[bytes] -> (data u8, offsets u64, lengths u64), back to back."""
    lengths = np.array([len(m) for m in messages], dtype=np.uint64)
    offsets = np.zeros(len(messages), dtype=np.uint64)
    if len(messages):
        offsets[1:] = np.cumsum(lengths)[:-1]
    data = np.frombuffer(b"".join(bytes(m) for m in messages), dtype=np.uint8).copy()
    if data.size == 0:
        data = np.zeros(1, dtype=np.uint8)
    return data, offsets, lengths


class Oracle:
    def __init__(self):
        if not ORACLE_SO.exists():
            build()
        self.lib = lib = C.CDLL(str(ORACLE_SO))
        lib.ko_permute_1600.argtypes = [u64p]
        lib.ko_permute_1600.restype = None
        lib.ko_rate_bytes.argtypes = [C.c_int]
        lib.ko_rate_bytes.restype = C.c_uint
        lib.ko_digest_bytes.argtypes = [C.c_int, C.c_uint64]
        lib.ko_digest_bytes.restype = C.c_uint64
        lib.ko_hash_one.argtypes = [C.c_int, C.c_uint64, u8p, C.c_uint64, u8p]
        lib.ko_hash_one.restype = C.c_int
        lib.ko_hash_batch.argtypes = [C.c_int, u8p, u64p, u64p, C.c_uint64, C.c_uint64,
                                      C.c_uint64, u8p, C.c_uint]
        lib.ko_hash_batch.restype = C.c_int
        lib.ko_generate_workload.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u8p]
        lib.ko_generate_workload.restype = C.c_uint64
        lib.ko_testrng_below.argtypes = [u64p, C.c_uint64]
        lib.ko_testrng_below.restype = C.c_uint64
        lib.ko_testrng_bytes.argtypes = [u64p, u8p, C.c_uint64]
        lib.ko_testrng_bytes.restype = None

    def permute(self, lanes: np.ndarray) -> np.ndarray:
        a = np.array(lanes, dtype=np.uint64).reshape(25).copy()
        self.lib.ko_permute_1600(_ptr(a, u64p))
        return a

    def rate_bytes(self, algorithm: int) -> int:
        return int(self.lib.ko_rate_bytes(algorithm))

    def digest_bytes(self, algorithm: int, xof_bits: int = 0) -> int:
        return int(self.lib.ko_digest_bytes(algorithm, xof_bits))

    def hash_one(self, algorithm: int, message: bytes, xof_bits: int = 0) -> bytes:
        msg = _as_u8(message)
        n = self.digest_bytes(algorithm, xof_bits)
        out = np.zeros(max(n, 1), dtype=np.uint8)
        src = msg if msg.size else np.zeros(1, dtype=np.uint8)
        rc = self.lib.ko_hash_one(algorithm, xof_bits, _ptr(src, u8p), msg.size, _ptr(out, u8p))
        if rc != 0:
            raise ValueError("oracle: invalid argument")
        return out[:n].tobytes()

    def hash_batch(self, algorithm: int, data, offsets=None, lengths=None, *,
                   fixed_len: int = 0, count: int | None = None, xof_bits: int = 0,
                   workers: int = 1) -> np.ndarray:
        data = _as_u8(data)
        if lengths is not None:
            lengths = np.ascontiguousarray(lengths, dtype=np.uint64)
            offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
            count = len(lengths)
        assert count is not None
        n = self.digest_bytes(algorithm, xof_bits)
        out = np.zeros((count, n), dtype=np.uint8)
        rc = self.lib.ko_hash_batch(algorithm, _ptr(data, u8p), _ptr(offsets, u64p),
                                    _ptr(lengths, u64p), fixed_len, count, xof_bits,
                                    _ptr(out.reshape(-1) if out.size else np.zeros(1, np.uint8), u8p),
                                    workers)
        if rc != 0:
            raise ValueError("oracle: invalid argument")
        return out

    def generate_workload(self, total_bytes: int, message_size: int, seed: int = 1) -> np.ndarray:
        count = total_bytes // message_size
        out = np.zeros(count * message_size, dtype=np.uint8)
        got = self.lib.ko_generate_workload(seed, total_bytes, message_size, _ptr(out, u8p))
        assert got == count
        return out

    # --- reference test RNG (tests/test_util.hpp:14-35) -------------------
    class TestRng:
        def __init__(self, lib, seed: int):
            self.lib = lib
            self.state = C.c_uint64(seed)

        def below(self, n: int) -> int:
            return int(self.lib.ko_testrng_below(C.byref(self.state), n))

        def random_bytes(self, n: int) -> bytes:
            out = np.zeros(max(n, 1), dtype=np.uint8)
            self.lib.ko_testrng_bytes(C.byref(self.state), _ptr(out, u8p), n)
            return out[:n].tobytes()

    def test_rng(self, seed: int) -> "Oracle.TestRng":
        return Oracle.TestRng(self.lib, seed)


class Reference:
    """The compiled reference (kind = "reference" CPU baseline)."""

    @staticmethod
    def available(hash_into: bool = False) -> bool:
        return (REF_HASHINTO_SO if hash_into else REF_SO).exists()

    def __init__(self, hash_into: bool = False):
        """hash_into=True loads the build whose parallel branch hashes into the pre-sized
        slots (oracle/ref_prelude.hpp): the reference's best case as a CPU baseline."""
        so = REF_HASHINTO_SO if hash_into else REF_SO
        if not so.exists():
            raise FileNotFoundError(f"{so} not built (needs /root/reference; see oracle/Makefile)")
        self.lib = lib = C.CDLL(str(so))
        lib.ref_batch_create.argtypes = [C.c_int, u8p, u64p, u64p, C.c_uint64, C.c_uint64, C.c_uint64]
        lib.ref_batch_create.restype = C.c_void_p
        lib.ref_batch_run.argtypes = [C.c_void_p, C.c_int, C.c_uint, C.c_uint64, u8p,
                                      C.POINTER(C.c_double)]
        lib.ref_batch_run.restype = C.c_int
        lib.ref_batch_destroy.argtypes = [C.c_void_p]
        lib.ref_batch_destroy.restype = None
        lib.ref_hash_batch.argtypes = [C.c_int, u8p, u64p, u64p, C.c_uint64, C.c_uint64,
                                       C.c_uint64, u8p, C.c_int, C.c_uint, C.c_uint64,
                                       C.POINTER(C.c_double)]
        lib.ref_hash_batch.restype = C.c_int
        lib.ref_one_shot.argtypes = [C.c_int, u8p, C.c_uint64, C.c_uint64, u8p]
        lib.ref_one_shot.restype = C.c_int
        lib.ref_permute_1600.argtypes = [u64p]
        lib.ref_permute_1600.restype = None
        lib.ref_generate_workload.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u8p]
        lib.ref_generate_workload.restype = C.c_uint64
        lib.ref_hardware_workers.argtypes = []
        lib.ref_hardware_workers.restype = C.c_uint

    def permute(self, lanes) -> np.ndarray:
        a = np.array(lanes, dtype=np.uint64).reshape(25).copy()
        self.lib.ref_permute_1600(_ptr(a, u64p))
        return a

    def hardware_workers(self) -> int:
        return int(self.lib.ref_hardware_workers())

    def one_shot(self, algorithm: int, message: bytes, xof_bits: int = 0) -> bytes:
        msg = _as_u8(message)
        n = (xof_bits + 7) // 8 if algorithm >= 4 else (28, 32, 48, 64)[algorithm]
        out = np.zeros(max(n, 1), dtype=np.uint8)
        src = msg if msg.size else np.zeros(1, dtype=np.uint8)
        rc = self.lib.ref_one_shot(algorithm, _ptr(src, u8p), msg.size, xof_bits, _ptr(out, u8p))
        if rc == 1:
            raise ValueError("reference: std::invalid_argument")
        if rc != 0:
            raise RuntimeError("reference: exception")
        return out[:n].tobytes()

    def hash_batch(self, algorithm: int, data, offsets=None, lengths=None, *,
                   fixed_len: int = 0, count: int | None = None, xof_bits: int = 0,
                   parallel: bool = True, workers: int = 0, chunk: int = 0,
                   return_elapsed: bool = False):
        data = _as_u8(data)
        if lengths is not None:
            lengths = np.ascontiguousarray(lengths, dtype=np.uint64)
            offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
            count = len(lengths)
        assert count is not None
        n = (xof_bits + 7) // 8 if algorithm >= 4 else (28, 32, 48, 64)[algorithm]
        out = np.zeros((count, n), dtype=np.uint8)
        elapsed = C.c_double(0)
        flat = out.reshape(-1) if out.size else np.zeros(1, np.uint8)
        rc = self.lib.ref_hash_batch(algorithm, _ptr(data, u8p), _ptr(offsets, u64p),
                                     _ptr(lengths, u64p), fixed_len, count, xof_bits,
                                     _ptr(flat, u8p), 1 if parallel else 0, workers, chunk,
                                     C.byref(elapsed))
        if rc == 1:
            raise ValueError("reference: std::invalid_argument")
        if rc != 0:
            raise RuntimeError("reference: exception")
        return (out, elapsed.value) if return_elapsed else out

    class Batch:
        """A HashBatch kept alive across timed runs (vector<vector> built once)."""

        def __init__(self, ref: "Reference", algorithm, data, fixed_len, count, xof_bits=0):
            self.ref = ref
            data = _as_u8(data)
            self.handle = ref.lib.ref_batch_create(algorithm, _ptr(data, u8p), None, None,
                                                   fixed_len, count, xof_bits)
            if not self.handle:
                raise MemoryError("reference: batch allocation failed")

        def run(self, parallel=True, workers=0, chunk=0) -> float:
            elapsed = C.c_double(0)
            rc = self.ref.lib.ref_batch_run(self.handle, 1 if parallel else 0, workers, chunk,
                                            None, C.byref(elapsed))
            if rc != 0:
                raise RuntimeError(f"reference: hash_batch failed ({rc})")
            return elapsed.value

        def close(self):
            if self.handle:
                self.ref.lib.ref_batch_destroy(self.handle)
                self.handle = None

        def __del__(self):
            self.close()

    def generate_workload(self, total_bytes: int, message_size: int, seed: int = 1) -> np.ndarray:
        count = total_bytes // message_size
        out = np.zeros(count * message_size, dtype=np.uint8)
        got = self.lib.ref_generate_workload(seed, total_bytes, message_size, _ptr(out, u8p))
        assert got == count
        return out
