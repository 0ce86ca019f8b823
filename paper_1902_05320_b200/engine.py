"""ctypes binding of libb200sha3.so (the C ABI in include/b200sha3.h).

Mirrors the reference's batch surface (proj/core/include/sha3/batch.hpp:23-65)
over packed buffers:

    Engine().hash_batch(algorithm, data, offsets, lengths, xof_output_bits=0)
    Engine().hash_fixed(algorithm, data, msg_len, count, xof_output_bits=0)

``data`` / ``offsets`` / ``lengths`` may be numpy arrays (host entry points:
the library copies to the GPU, hashes, copies back) or CUDA torch tensors
(device entry points: asynchronous on the current torch stream, digests stay
in HBM).  Errors follow the reference: a bad algorithm or an XOF without an
output length raises ``ValueError`` (std::invalid_argument, batch.cpp:66-68)
before any work; anything CUDA raises ``EngineError``.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

ALGORITHMS = ("sha3_224", "sha3_256", "sha3_384", "sha3_512", "shake128", "shake256")

_HERE = pathlib.Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libb200sha3.so"

OK, ERR_INVALID_ARGUMENT, ERR_CUDA, ERR_UNSUPPORTED, ERR_STATE = 0, 1, 2, 3, 4
FLAG_NO_BUCKETING, FLAG_NO_PIPELINE, FLAG_NO_WARP_KERNEL = 1, 2, 4
KERNEL_AUTO, KERNEL_GENERIC, KERNEL_ONEBLOCK, KERNEL_LANESPLIT, KERNEL_STAGED, KERNEL_WARP, KERNEL_PAIR = 0, 1, 2, 3, 4, 5, 6
KERNEL_FEWBLOCK = 7

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class EngineError(RuntimeError):
    """CUDA failure or unsupported batch shape reported by the library."""


class EngineStateError(RuntimeError):
    """Incremental API used out of order (std::logic_error in the reference)."""


class _Config(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("device", C.c_int32), ("stream", C.c_void_p),
                ("flags", C.c_uint32), ("kernel", C.c_int32), ("unroll", C.c_int32),
                ("fma_preset", C.c_int32), ("block_threads", C.c_int32),
                ("device_ms", C.POINTER(C.c_double)), ("kernel_launches", u32p)]


def library_path() -> pathlib.Path:
    return _LIB_PATH


def library_info() -> dict:
    """Provenance of the loaded library for reports: path, version string (compiler and build
    time, from the library itself), size, modification time and a CRC-32 of the file."""
    import time
    import zlib
    raw = _LIB_PATH.read_bytes()
    stat = _LIB_PATH.stat()
    return {"path": str(_LIB_PATH), "version": _library().b200sha3_version().decode(), "bytes": len(raw),
            "mtime_utc": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime(stat.st_mtime)),
            "crc32": f"{zlib.crc32(raw):08x}"}


def algorithm_id(algorithm) -> int:
    if isinstance(algorithm, str):
        name = algorithm.lower().replace("-", "_")
        if name not in ALGORITHMS:
            raise ValueError(f"unknown algorithm {algorithm!r}")
        return ALGORITHMS.index(name)
    return int(algorithm)


def _load() -> C.CDLL:
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(str(_LIB_PATH))
    cfgp = C.POINTER(_Config)
    lib.b200sha3_digest_bytes.argtypes = [C.c_int, C.c_uint64]
    lib.b200sha3_digest_bytes.restype = C.c_uint64
    lib.b200sha3_rate_bytes.argtypes = [C.c_int]
    lib.b200sha3_rate_bytes.restype = C.c_uint32
    lib.b200sha3_permutations.argtypes = [C.c_int, C.c_uint64, C.c_uint64]
    lib.b200sha3_permutations.restype = C.c_uint64
    lib.b200sha3_selected_kernel.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64]
    lib.b200sha3_selected_kernel.restype = C.c_char_p
    lib.b200sha3_strerror.argtypes = [C.c_int]
    lib.b200sha3_strerror.restype = C.c_char_p
    lib.b200sha3_last_cuda_error.argtypes = []
    lib.b200sha3_last_cuda_error.restype = C.c_char_p
    lib.b200sha3_version.argtypes = []
    lib.b200sha3_version.restype = C.c_char_p
    for name in ("b200sha3_hash_batch", "b200sha3_hash_batch_device"):
        fn = getattr(lib, name)
        fn.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64,
                       C.c_void_p, cfgp]
        fn.restype = C.c_int
    for name in ("b200sha3_hash_fixed", "b200sha3_hash_fixed_device"):
        fn = getattr(lib, name)
        fn.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p, cfgp]
        fn.restype = C.c_int
    lib.b200sha3_generate_workload_device.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64,
                                                      C.c_uint64, C.c_uint64, C.c_void_p, cfgp]
    lib.b200sha3_generate_workload_device.restype = C.c_int
    lib.b200sha3_generate_lengths_device.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64,
                                                     C.c_uint64, C.c_uint64, C.c_void_p, cfgp]
    lib.b200sha3_generate_lengths_device.restype = C.c_int
    lib.b200sha3_fill_messages_device.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p,
                                                  C.c_void_p, C.c_void_p, cfgp]
    lib.b200sha3_fill_messages_device.restype = C.c_int
    lib.b200sha3_permute_device.argtypes = [C.c_void_p, C.c_uint64, cfgp]
    lib.b200sha3_permute_device.restype = C.c_int
    lib.b200sha3_bucket_order_device.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, cfgp]
    lib.b200sha3_bucket_order_device.restype = C.c_int
    lib.b200sha3_pinned_alloc.argtypes = [C.c_uint64, C.POINTER(C.c_void_p)]
    lib.b200sha3_pinned_alloc.restype = C.c_int
    lib.b200sha3_pinned_free.argtypes = [C.c_void_p]
    lib.b200sha3_pinned_free.restype = C.c_int
    lib.b200sha3_states_create.argtypes = [C.c_int, C.c_uint64, cfgp, C.POINTER(C.c_void_p)]
    lib.b200sha3_states_create.restype = C.c_int
    lib.b200sha3_states_destroy.argtypes = [C.c_void_p]
    lib.b200sha3_states_destroy.restype = C.c_int
    lib.b200sha3_states_reset.argtypes = [C.c_void_p, cfgp]
    lib.b200sha3_states_reset.restype = C.c_int
    lib.b200sha3_states_update_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, cfgp]
    lib.b200sha3_states_update_device.restype = C.c_int
    lib.b200sha3_states_update_fixed_device.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, cfgp]
    lib.b200sha3_states_update_fixed_device.restype = C.c_int
    lib.b200sha3_states_finish_device.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, cfgp]
    lib.b200sha3_states_finish_device.restype = C.c_int
    lib.b200sha3_states_squeeze_device.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, cfgp]
    lib.b200sha3_states_squeeze_device.restype = C.c_int
    lib.b200sha3_probe_pipe.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), cfgp]
    lib.b200sha3_probe_pipe.restype = C.c_int
    return lib


_lib = None


def _library() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def digest_bytes(algorithm, xof_output_bits: int = 0) -> int:
    return int(_library().b200sha3_digest_bytes(algorithm_id(algorithm), xof_output_bits))


def rate_bytes(algorithm) -> int:
    return int(_library().b200sha3_rate_bytes(algorithm_id(algorithm)))


def permutations(algorithm, msg_len: int, xof_output_bits: int = 0) -> int:
    return int(_library().b200sha3_permutations(algorithm_id(algorithm), msg_len, xof_output_bits))


def selected_kernel(algorithm, msg_len: int | None, xof_output_bits: int = 0, count: int = 1 << 24) -> str:
    """Name of the kernel KERNEL_AUTO picks for `count` equal-length messages of msg_len bytes
    (None: a variable-length batch) on aligned buffers."""
    n = (1 << 64) - 1 if msg_len is None else msg_len
    return _library().b200sha3_selected_kernel(algorithm_id(algorithm), n, count, xof_output_bits).decode()


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


class Engine:
    """One configuration of the engine (the analogue of sha3::EngineConfig)."""

    def __init__(self, device: int | None = None, *, kernel: int = KERNEL_AUTO, unroll: int = 0,
                 fma_preset: int = -1, block_threads: int = 0, flags: int = 0):
        self.lib = _library()
        self.device = device
        self.kernel = kernel
        self.unroll = unroll
        self.fma_preset = fma_preset
        self.block_threads = block_threads
        self.flags = flags
        self.last_device_ms = 0.0
        self.last_kernel_launches = 0
        self.total_kernel_launches = 0

    # -- plumbing ---------------------------------------------------------
    def _config(self, stream_ptr, timed: bool):
        ms = C.c_double(0.0)
        launches = C.c_uint32(0)
        cfg = _Config(C.sizeof(_Config), -1 if self.device is None else int(self.device),
                      stream_ptr, self.flags, self.kernel, self.unroll, self.fma_preset,
                      self.block_threads, C.pointer(ms) if timed else None, C.pointer(launches))
        return cfg, ms, launches

    def _check(self, rc: int):
        if rc == OK:
            return
        if rc == ERR_INVALID_ARGUMENT:
            raise ValueError("b200sha3: invalid argument (bad algorithm id, or an XOF variant "
                             "without xof_output_bits)")
        if rc == ERR_STATE:
            raise EngineStateError("b200sha3: incremental API used out of order")
        detail = self.lib.b200sha3_last_cuda_error().decode()
        raise EngineError(f"b200sha3: {self.lib.b200sha3_strerror(rc).decode()}: {detail}")

    def _finish(self, rc, ms, launches, timed):
        self._check(rc)
        self.last_device_ms = ms.value if timed else 0.0
        self.last_kernel_launches = launches.value
        self.total_kernel_launches += launches.value

    @staticmethod
    def _torch_stream():
        import torch
        return torch.cuda.current_stream().cuda_stream

    @staticmethod
    def _np(a, dtype):
        return np.ascontiguousarray(a, dtype=dtype).reshape(-1)

    # -- the hot path -----------------------------------------------------
    def hash_fixed(self, algorithm, data, msg_len: int, count: int, xof_output_bits: int = 0,
                   out=None, timed: bool = False):
        """Equal-length messages packed back to back.  Returns (count, digest_bytes) uint8."""
        alg = algorithm_id(algorithm)
        nbytes = int(self.lib.b200sha3_digest_bytes(alg, xof_output_bits)) if 0 <= alg <= 5 else 0
        if _is_torch(data):
            import torch
            assert data.is_cuda and data.dtype == torch.uint8 and data.is_contiguous()
            if out is None:
                out = torch.empty((count, nbytes), dtype=torch.uint8, device=data.device)
            cfg, ms, launches = self._config(self._torch_stream(), timed)
            rc = self.lib.b200sha3_hash_fixed_device(alg, data.data_ptr(), msg_len, count,
                                                     xof_output_bits, out.data_ptr(), C.byref(cfg))
        else:
            data = self._np(data, np.uint8)
            if out is None:
                out = np.empty((count, nbytes), dtype=np.uint8)
            cfg, ms, launches = self._config(None, timed)
            rc = self.lib.b200sha3_hash_fixed(alg, data.ctypes.data, msg_len, count,
                                              xof_output_bits, out.ctypes.data, C.byref(cfg))
        self._finish(rc, ms, launches, timed)
        return out

    def hash_fixed_ptr(self, algorithm, data_ptr: int, msg_len: int, count: int, out_ptr: int,
                       xof_output_bits: int = 0, timed: bool = False):
        """Host entry on raw host addresses (pinned staging buffers in bench.py)."""
        cfg, ms, launches = self._config(None, timed)
        rc = self.lib.b200sha3_hash_fixed(algorithm_id(algorithm), data_ptr, msg_len, count,
                                          xof_output_bits, out_ptr, C.byref(cfg))
        self._finish(rc, ms, launches, timed)

    def hash_batch(self, algorithm, data, offsets, lengths, xof_output_bits: int = 0, out=None,
                   timed: bool = False):
        """Variable-length messages: message i is data[offsets[i] : offsets[i]+lengths[i]]."""
        alg = algorithm_id(algorithm)
        nbytes = int(self.lib.b200sha3_digest_bytes(alg, xof_output_bits)) if 0 <= alg <= 5 else 0
        if _is_torch(data):
            import torch
            count = int(lengths.numel())
            assert data.is_cuda and data.dtype == torch.uint8
            assert offsets.dtype in (torch.int64, torch.uint64) and lengths.dtype == offsets.dtype
            if out is None:
                out = torch.empty((count, nbytes), dtype=torch.uint8, device=data.device)
            cfg, ms, launches = self._config(self._torch_stream(), timed)
            rc = self.lib.b200sha3_hash_batch_device(alg, data.data_ptr(), offsets.data_ptr(),
                                                     lengths.data_ptr(), count, xof_output_bits,
                                                     out.data_ptr(), C.byref(cfg))
        else:
            data = self._np(data, np.uint8)
            offsets = self._np(offsets, np.uint64)
            lengths = self._np(lengths, np.uint64)
            count = len(lengths)
            if out is None:
                out = np.empty((count, nbytes), dtype=np.uint8)
            cfg, ms, launches = self._config(None, timed)
            rc = self.lib.b200sha3_hash_batch(alg, data.ctypes.data if data.size else None,
                                              offsets.ctypes.data if count else None,
                                              lengths.ctypes.data if count else None, count,
                                              xof_output_bits,
                                              out.ctypes.data if out.size else None, C.byref(cfg))
        self._finish(rc, ms, launches, timed)
        return out

    def hash_messages(self, algorithm, messages, xof_output_bits: int = 0):
        """list[bytes] -> list[bytes]; the HashBatch -> BatchResult shape of the reference."""
        lengths = np.array([len(m) for m in messages], dtype=np.uint64)
        offsets = np.zeros(len(messages), dtype=np.uint64)
        if len(messages):
            offsets[1:] = np.cumsum(lengths)[:-1]
        blob = b"".join(bytes(m) for m in messages)
        data = np.frombuffer(blob, dtype=np.uint8) if blob else np.zeros(1, dtype=np.uint8)
        out = self.hash_batch(algorithm, data, offsets, lengths, xof_output_bits)
        return [out[i].tobytes() for i in range(len(messages))]

    # -- harness helpers --------------------------------------------------
    def generate_workload(self, total_bytes: int, message_size: int, *, seed: int = 1,
                          first_message: int = 0, count: int | None = None, device=None):
        """Device version of generate_workload (workload.cpp:16-47); returns a CUDA uint8 tensor."""
        import torch
        if count is None:
            count = total_bytes // message_size
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        out = torch.empty(max(count * message_size, 16), dtype=torch.uint8, device=dev)
        cfg, ms, launches = self._config(self._torch_stream(), False)
        rc = self.lib.b200sha3_generate_workload_device(seed, total_bytes, message_size,
                                                        first_message, count, out.data_ptr(),
                                                        C.byref(cfg))
        self._check(rc)
        self.total_kernel_launches += 1 if count else 0   # harness kernels count too (ncu sees them)
        return out[:count * message_size]

    def generate_lengths(self, count: int, min_len: int, max_len: int, *, seed_len: int = 2,
                         first_message: int = 0):
        import torch
        out = torch.empty(max(count, 1), dtype=torch.int64, device="cuda")
        cfg, _, _ = self._config(self._torch_stream(), False)
        rc = self.lib.b200sha3_generate_lengths_device(seed_len, min_len, max_len, first_message,
                                                       count, out.data_ptr(), C.byref(cfg))
        self._check(rc)
        self.total_kernel_launches += 1 if count else 0
        return out[:count]

    def fill_messages(self, data, offsets, lengths, *, seed: int = 1, first_message: int = 0):
        cfg, _, _ = self._config(self._torch_stream(), False)
        rc = self.lib.b200sha3_fill_messages_device(seed, first_message, int(lengths.numel()),
                                                    offsets.data_ptr(), lengths.data_ptr(),
                                                    data.data_ptr(), C.byref(cfg))
        self._check(rc)
        self.total_kernel_launches += 1 if lengths.numel() else 0

    def permute_states(self, states):
        """In-place Keccak-f[1600] on a (n, 25) int64/uint64 CUDA tensor."""
        cfg, _, _ = self._config(self._torch_stream(), False)
        rc = self.lib.b200sha3_permute_device(states.data_ptr(), states.shape[0], C.byref(cfg))
        self._check(rc)
        self.total_kernel_launches += 1 if states.shape[0] else 0
        return states

    def bucket_order(self, algorithm, lengths):
        import torch
        order = torch.empty(max(int(lengths.numel()), 1), dtype=torch.int32, device=lengths.device)
        cfg, _, _ = self._config(self._torch_stream(), False)
        rc = self.lib.b200sha3_bucket_order_device(algorithm_id(algorithm), lengths.data_ptr(),
                                                   int(lengths.numel()), order.data_ptr(),
                                                   C.byref(cfg))
        self._check(rc)
        return order[:lengths.numel()]

    def probe_pipe(self, mix: int):
        """(thread-instructions per second, SM clock in Hz) for one instruction mix."""
        rate, hz = C.c_double(0), C.c_double(0)
        cfg, _, _ = self._config(None, False)
        rc = self.lib.b200sha3_probe_pipe(mix, C.byref(rate), C.byref(hz), C.byref(cfg))
        self._check(rc)
        return rate.value, hz.value


class BatchHasher:
    """`count` incremental hashers resident in HBM -- the batch analogue of sha3::Hasher
    (proj/core/include/sha3/sha3.hpp:66-86): update() any number of times, then digest()
    (hash variants) or finish() + read() (XOF variants).  CUDA torch tensors in and out."""

    def __init__(self, algorithm, count: int, engine: Engine | None = None):
        self.engine = engine or Engine()
        self.algorithm = algorithm_id(algorithm)
        self.count = count
        self._handle = C.c_void_p()
        cfg, _, _ = self.engine._config(Engine._torch_stream(), False)
        self.engine._check(self.engine.lib.b200sha3_states_create(self.algorithm, count, C.byref(cfg),
                                                                  C.byref(self._handle)))

    def close(self):
        if self._handle:
            self.engine.lib.b200sha3_states_destroy(self._handle)
            self._handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _cfg(self):
        return self.engine._config(Engine._torch_stream(), False)[0]

    def update(self, data, offsets=None, lengths=None, chunk_len: int | None = None):
        cfg = self._cfg()
        if chunk_len is not None:
            rc = self.engine.lib.b200sha3_states_update_fixed_device(self._handle, data.data_ptr(), chunk_len,
                                                                     C.byref(cfg))
        else:
            rc = self.engine.lib.b200sha3_states_update_device(self._handle, data.data_ptr(),
                                                               offsets.data_ptr(), lengths.data_ptr(),
                                                               C.byref(cfg))
        self.engine._check(rc)

    def _finish(self, bits: int):
        import torch
        nbytes = int(self.engine.lib.b200sha3_digest_bytes(self.algorithm, bits))
        out = torch.empty((self.count, nbytes), dtype=torch.uint8, device="cuda") if nbytes else None
        cfg = self._cfg()
        rc = self.engine.lib.b200sha3_states_finish_device(self._handle, bits,
                                                           out.data_ptr() if out is not None else None,
                                                           C.byref(cfg))
        self.engine._check(rc)
        return out

    def digest(self):
        """Hash variants: finalize, return (count, digest_bytes)."""
        if self.algorithm >= 4:
            raise EngineStateError("digest() is for fixed-output variants; use finish()/read()")
        return self._finish(0)

    def finish(self, xof_output_bits: int = 0):
        """XOF variants: close the input; optionally return the first ceil(bits/8) bytes."""
        if self.algorithm < 4:
            raise EngineStateError("finish()/read() is for XOF variants; use digest()")
        return self._finish(xof_output_bits)

    def read(self, nbytes: int):
        import torch
        out = torch.empty((self.count, nbytes), dtype=torch.uint8, device="cuda")
        cfg = self._cfg()
        self.engine._check(self.engine.lib.b200sha3_states_squeeze_device(self._handle, nbytes,
                                                                          out.data_ptr(), C.byref(cfg)))
        return out

    def reset(self):
        cfg = self._cfg()
        self.engine._check(self.engine.lib.b200sha3_states_reset(self._handle, C.byref(cfg)))


def splitmix64_at(seed, n):
    """numpy: output number n (1-based, array ok) of splitmix64 seeded with `seed`."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + np.asarray(n, dtype=np.uint64) * np.uint64(0x9e3779b97f4a7c15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
        return z ^ (z >> np.uint64(31))
