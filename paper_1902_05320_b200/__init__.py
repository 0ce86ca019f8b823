"""B200-native batch SHA-3 / SHAKE engine (the `sha3::hash_batch` hot path).

The product is the C-ABI shared library ``libb200sha3.so`` (hand-written
sm_100a kernels; see ``include/b200sha3.h``) plus the C++ adapter in
``include/b200sha3/batch.hpp``.  This Python package is only the thin ctypes
binding that the tests and ``bench.py`` drive it with; PyTorch supplies device
memory, streams and ``torch.distributed`` and nothing else.

There is no CPU fallback: importing ``engine`` without the built library, or
calling it without a CUDA device, raises.
"""
from .engine import (ALGORITHMS, BatchHasher, Engine, EngineError, EngineStateError,  # noqa: F401
                     algorithm_id, digest_bytes, library_info, library_path, permutations, rate_bytes,
                     selected_kernel)
