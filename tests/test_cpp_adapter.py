"""Builds and runs tests/cpp/test_batch_adapter (the reference's test_batch.cpp
hash_batch cases restated against the C++ adapter / sha3::hash_batch drop-in)."""
import pathlib
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
EXE = ROOT / "tests" / "cpp" / "test_batch_adapter"


def build():
    subprocess.run(["make", "-C", str(ROOT / "paper_1902_05320_b200" / "host")], check=True,
                   stdout=subprocess.DEVNULL)
    subprocess.run(["make", "-C", str(ROOT / "oracle"), "liboracle.so"], check=True,
                   stdout=subprocess.DEVNULL)
    subprocess.run(["make", "-C", str(ROOT / "tests" / "cpp")], check=True, stdout=subprocess.DEVNULL)


def test_adapter_cpu_only_cases():
    """XOF-without-length throws std::invalid_argument with the reference's message before
    any work; an empty batch gives an empty result -- no device needed."""
    build()
    out = subprocess.run([str(EXE), "--cpu-only"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout


@pytest.mark.gpu
def test_adapter_all_cases():
    build()
    out = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failures" in out.stdout


@pytest.mark.gpu
def test_reference_runner_on_our_backend():
    """Binding 2 of INTEGRATION.md, executed: the reference's unmodified run_benchmark /
    emit_csv / generate_workload, linked against our sha3::hash_batch instead of its
    batch.cpp (recipe: oracle/Makefile `runner`; source: tests/integration/ref_runner_main.cpp;
    built where /root/reference is mounted).  The binary also
    cross-checks 5000 digests against the reference's own CPU sha3_digest."""
    exe = ROOT / "oracle" / "_ref" / "ref_runner_on_b200"
    subprocess.run(["make", "-C", str(ROOT / "oracle"), "runner"], check=False,
                   stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    if not exe.exists():
        pytest.skip("integration binary not built (needs /root/reference at build time)")
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = out.stdout.strip().splitlines()
    assert lines[0] == "total_bytes,message_size,message_count,backend,time_seconds,throughput_bps,repeats"
    assert len(lines) == 5 and lines[1].startswith("64000,64,1000,")
    assert "5000/5000 digests equal" in lines[-1]


def _build_target(*args):
    return subprocess.run(["make", "-C", str(ROOT / "tests" / "cpp"), *args], capture_output=True, text=True)


@pytest.mark.parametrize("sanitizer", ["thread", "address"])
def test_adapter_scheduling_under_sanitizer(sanitizer):
    """The host-side pipeline of the C++ adapter (scan, chunk plan, pinned ring, pack / device-call /
    unpack tasks, speculative restart, failure propagation) under ThreadSanitizer / AddressSanitizer
    with the C ABI answered by a test double over the oracle (tests/cpp/fake_device_capi.cpp) and
    every plan size divided by 512, so ring wrap-around and multi-step resizes happen on small
    batches.  Random shapes, worker counts, device lists, concurrent callers, injected device
    failures; every digest is compared with the oracle.  No GPU involved."""
    subprocess.run(["make", "-C", str(ROOT / "oracle"), "liboracle.so"], check=True, stdout=subprocess.DEVNULL)
    built = _build_target(f"SAN={sanitizer}", f"fuzz_batch_adapter_{sanitizer}")
    if built.returncode != 0:
        pytest.skip(f"-fsanitize={sanitizer} runtime not available: {built.stderr[-200:]}")
    exe = ROOT / "tests" / "cpp" / f"fuzz_batch_adapter_{sanitizer}"
    out = subprocess.run([str(exe), "6", "5", "14"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert '"mismatching_batches": 0' in out.stdout
    assert "ThreadSanitizer" not in out.stderr and "AddressSanitizer" not in out.stderr


@pytest.mark.gpu
def test_adapter_fuzz_on_device():
    """The same randomized batches through the real device (libb200sha3.so), up to 2^19 messages so
    the thread pool, several chunks and the speculative equal-length plan are all taken."""
    build()
    assert _build_target("fuzz_batch_adapter").returncode == 0
    out = subprocess.run([str(ROOT / "tests" / "cpp" / "fuzz_batch_adapter"), "15", "7", "19"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert '"mismatching_batches": 0' in out.stdout
