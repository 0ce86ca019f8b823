"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/b200sha3.h declares, answers the pure queries, applies the
reference's validation order without a GPU, and fails loudly (no CPU fallback)
when asked to compute without one."""
import ctypes
import pathlib
import re

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "b200sha3.h").read_text()
    return sorted(set(re.findall(r"B200SHA3_API\s+[\w\s\*]+?\b(b200sha3_\w+)\s*\(", text)))


def test_header_declares_the_expected_entry_points():
    names = declared_symbols()
    for required in ("b200sha3_hash_batch", "b200sha3_hash_fixed", "b200sha3_hash_batch_device",
                     "b200sha3_hash_fixed_device", "b200sha3_digest_bytes", "b200sha3_strerror"):
        assert required in names
    assert len(names) >= 16


def test_library_exports_every_declared_symbol():
    from paper_1902_05320_b200 import library_path
    lib = ctypes.CDLL(str(library_path()))
    for name in declared_symbols():
        assert hasattr(lib, name), f"{name} declared in include/b200sha3.h but not exported"


def test_queries_match_the_variant_table():
    """proj/core/src/sha3.cpp:13-20 and batch.cpp:74-75."""
    import paper_1902_05320_b200 as eng
    assert [eng.rate_bytes(a) for a in range(6)] == [144, 136, 104, 72, 168, 136]
    assert [eng.digest_bytes(a, 999) for a in range(4)] == [28, 32, 48, 64]  # bits ignored for hashes
    assert eng.digest_bytes("shake128", 328) == 41 and eng.digest_bytes("shake256", 8) == 1
    assert eng.digest_bytes(6) == 0 and eng.rate_bytes(-1) == 0
    # permutations per message: floor(L/R) + 1 + extra squeeze blocks
    assert eng.permutations("sha3_256", 64) == 1
    assert eng.permutations("sha3_256", 136) == 2
    assert eng.permutations("sha3_256", 16384) == 121
    assert eng.permutations("sha3_512", 1024) == 15
    assert eng.permutations("shake128", 64, 4096) == 4
    assert eng.permutations("shake256", 64, 4096) == 4
    assert eng.algorithm_id("SHA3-256") == 1


def test_oracle_and_library_agree_on_queries(oracle):
    import paper_1902_05320_b200 as eng
    for a in range(6):
        assert eng.rate_bytes(a) == oracle.rate_bytes(a)
        for bits in (1, 8, 12, 328, 4096):
            assert eng.digest_bytes(a, bits) == oracle.digest_bytes(a, bits)


def test_validation_happens_before_any_work():
    """XOF without a length and bad ids are rejected up front (batch.cpp:66-68,
    test_batch.cpp:162-167) -- no CUDA needed to get the error."""
    from paper_1902_05320_b200 import Engine
    e = Engine()
    one = np.ones(1, dtype=np.uint8)
    with pytest.raises(ValueError):
        e.hash_fixed("shake256", one, 1, 1, xof_output_bits=0)
    with pytest.raises(ValueError):
        e.hash_batch(4, one, np.zeros(1, np.uint64), np.ones(1, np.uint64), xof_output_bits=0)
    with pytest.raises(ValueError):
        e.hash_fixed(6, one, 1, 1)
    with pytest.raises(ValueError):
        e.hash_fixed(-1, one, 1, 1)


def test_empty_batch_is_an_empty_result():
    """test_batch.cpp:113-117 -- also needs no device."""
    from paper_1902_05320_b200 import Engine
    e = Engine()
    assert e.hash_fixed("sha3_256", np.zeros(0, np.uint8), 64, 0).shape == (0, 32)
    out = e.hash_batch("shake128", np.zeros(0, np.uint8), np.zeros(0, np.uint64),
                       np.zeros(0, np.uint64), xof_output_bits=328)
    assert out.shape == (0, 41)
    assert e.hash_messages("sha3_512", []) == []


def test_no_cpu_fallback():
    """Without a CUDA device a compute call must raise, never return digests."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present; covered by the gpu tests")
    from paper_1902_05320_b200 import Engine, EngineError
    with pytest.raises(EngineError):
        Engine().hash_fixed("sha3_256", np.zeros(64, np.uint8), 64, 1)
    with pytest.raises(EngineError):
        Engine().hash_messages("sha3_256", [b"abc"])


def test_product_never_touches_the_oracle():
    """oracle/ is test infrastructure: nothing under the package, include/ or the
    C++ adapter may import, include or link it."""
    offenders = []
    for base in (ROOT / "paper_1902_05320_b200", ROOT / "include"):
        for path in base.rglob("*"):
            if path.suffix in {".py", ".cu", ".cuh", ".h", ".hpp", ".cpp", ".c"} or path.name == "Makefile":
                text = path.read_text(errors="ignore")
                if re.search(r"oracle|keccak_oracle|libsha3kit_ref|/root/reference", text):
                    offenders.append(str(path.relative_to(ROOT)))
    assert offenders == []


def test_misc_queries_without_a_device():
    import ctypes as C
    from paper_1902_05320_b200 import library_path
    lib = C.CDLL(str(library_path()))
    lib.b200sha3_version.restype = C.c_char_p
    lib.b200sha3_strerror.restype = C.c_char_p
    lib.b200sha3_strerror.argtypes = [C.c_int]
    assert b"sm_100a" in lib.b200sha3_version()
    assert lib.b200sha3_device_count() >= 0
    texts = {lib.b200sha3_strerror(i) for i in range(5)}
    assert len(texts) == 5 and b"unknown status" not in texts
    assert lib.b200sha3_strerror(99) == b"unknown status"
    # handles: bad algorithm is rejected before CUDA is touched; NULL handle calls are safe
    handle = C.c_void_p()
    lib.b200sha3_states_create.argtypes = [C.c_int, C.c_uint64, C.c_void_p, C.POINTER(C.c_void_p)]
    assert lib.b200sha3_states_create(7, 4, None, C.byref(handle)) == 1 and not handle.value
    lib.b200sha3_states_destroy.argtypes = [C.c_void_p]
    assert lib.b200sha3_states_destroy(None) == 0


def test_short_config_struct_is_honoured():
    """b200sha3_config::struct_size is the size the CALLER was built with: fields beyond it are
    never read.  A caller with a struct that ends before the two result pointers leaves garbage
    there; the library must not write through it (count == 0 returns before any CUDA call)."""
    from paper_1902_05320_b200.engine import _Config, _library
    lib = _library()
    cfg = _Config()
    ctypes.memset(ctypes.byref(cfg), 0xEE, ctypes.sizeof(cfg))   # every later field: garbage
    cfg.struct_size = _Config.device_ms.offset                   # an older, shorter struct
    cfg.device, cfg.stream, cfg.flags, cfg.kernel = -1, None, 0, 0
    cfg.unroll, cfg.fma_preset, cfg.block_threads = 0, -1, 0
    assert lib.b200sha3_hash_fixed_device(1, None, 64, 0, 0, None, ctypes.byref(cfg)) == 0
    assert lib.b200sha3_hash_batch(1, None, None, None, 0, 0, None, ctypes.byref(cfg)) == 0
    # struct_size 0 means "this version": the pointers are used
    ms, launches = ctypes.c_double(7.0), ctypes.c_uint32(7)
    cfg.struct_size = 0
    cfg.device_ms, cfg.kernel_launches = ctypes.pointer(ms), ctypes.pointer(launches)
    assert lib.b200sha3_hash_fixed_device(1, None, 64, 0, 0, None, ctypes.byref(cfg)) == 0
    assert ms.value == 0.0 and launches.value == 0


def test_selected_kernel_names():
    """Which kernel KERNEL_AUTO runs per shape (reports only; no GPU needed to ask)."""
    from paper_1902_05320_b200 import selected_kernel
    assert selected_kernel("sha3_256", 64) == "hash_oneblock_kernel<17,8,8>"
    assert selected_kernel("sha3_256", 10) == "hash_short_fixed_kernel<17,8>"
    assert selected_kernel("sha3_512", 1024) == "hash_fewblock_kernel<9,128,16>"  # static multi-block shape
    assert selected_kernel("sha3_512", 1032) == "hash_manyblock_kernel<9,16>"     # any whole number of lanes >= rate
    assert selected_kernel("sha3_512", 1030) == "hash_generic_kernel<9>"
    assert selected_kernel("shake256", 64, 4096) == "hash_fewblock_kernel<17,8,128>"
    assert selected_kernel("shake128", 64, 1023) == "hash_generic_kernel<21>"     # odd bits: masked tail
    assert selected_kernel("shake128", 64, 1024) == "hash_oneblock_kernel<21,8,32>"
    assert selected_kernel("sha3_256", None) == "bucket_order + hash_ragged_kernel<17,8>"
    assert selected_kernel("shake256", None, 4099) == "bucket_order + hash_generic_kernel<17>"
    assert selected_kernel(9, 64) == ""
    # few multi-block messages: one warp per message
    assert selected_kernel("sha3_256", 1 << 20, count=1024) == "hash_warp_kernel"
    assert selected_kernel("sha3_256", None, count=100) == "hash_warp_kernel"
    assert selected_kernel("sha3_256", 64, count=100) == "hash_oneblock_kernel<17,8,8>"   # single block
    assert selected_kernel("sha3_256", 1 << 20, count=1 << 14) == "hash_manyblock_kernel<17,8>"
    assert selected_kernel("sha3_256", (1 << 20) + 1, count=1 << 14) == "hash_generic_kernel<17>"
