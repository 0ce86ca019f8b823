"""Shared fixtures.  `-m "not gpu"` runs on the CPU-only build container,
`-m gpu` on a B200 box (no /root/reference there: golden vectors come from
tests/golden/, the compiled reference from the prebuilt oracle/_ref/)."""
import json
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"
REFERENCE_ROOT = pathlib.Path("/root/reference")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def load_kat_file(path):
    """-> (algorithm id, output bits, [(message bytes, digest bytes)])"""
    lines = path.read_text().splitlines()
    header = dict(tok.split("=") for tok in lines[0].lstrip("# ").split())
    vectors = []
    for line in lines[1:]:
        nbits, msg, md = line.split()
        m = b"" if msg == "-" else bytes.fromhex(msg)
        assert len(m) * 8 == int(nbits)
        vectors.append((m, bytes.fromhex(md)))
    assert len(vectors) == int(header["vectors"])
    return int(header["algorithm"]), int(header["output_bits"]), vectors


def all_kat_files():
    return sorted(GOLDEN.glob("*.kat"))


@pytest.fixture(scope="session")
def inline_kats():
    return json.loads((GOLDEN / "inline_kats.json").read_text())


@pytest.fixture(scope="session")
def oracle():
    from oracle.binding import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The compiled reference, or skip when oracle/_ref was never built."""
    from oracle.binding import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref/libsha3kit_ref.so not built (needs /root/reference)")
    return Reference()


@pytest.fixture(scope="session")
def engine():
    """The product default (KERNEL_AUTO: small multi-block batches take the warp-per-state
    kernel, everything else one message per thread)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1902_05320_b200 import Engine
    return Engine()


@pytest.fixture(scope="session")
def big_engine():
    """The product default again, under the name the full-size tests ask for (test modules that
    parametrize `engine` over kernel selections leave these tests alone)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_1902_05320_b200 import Engine
    return Engine()


def xof_bits_for(algorithm, out_bits):
    return out_bits if algorithm >= 4 else 0


def reference_style_batch(oracle, seed, count, max_len):
    """random_batch of proj/tests/test_batch.cpp:15-22: per message one below(max_len+1)
    draw for the length, then one draw per byte (tests/test_util.hpp:29-35)."""
    rng = oracle.test_rng(seed)
    return rng, [rng.random_bytes(rng.below(max_len + 1)) for _ in range(count)]
