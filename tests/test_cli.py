"""b200sha3cli: the `sha3cli bench` / `sha3cli vectors` callers of the hot path on the GPU
backend.  Response files are re-emitted from tests/golden/*.kat
in the reference's .rsp syntax (proj/tools/sha3cli/vectors.hpp:42-45)."""
import csv
import pathlib
import subprocess

import pytest

from conftest import GOLDEN, load_kat_file

ROOT = pathlib.Path(__file__).resolve().parent.parent
CLI = ROOT / "paper_1902_05320_b200" / "b200sha3cli"


@pytest.fixture(scope="module")
def cli():
    subprocess.run(["make", "-C", str(ROOT / "paper_1902_05320_b200" / "host")], check=True,
                   stdout=subprocess.DEVNULL)
    return CLI


def write_rsp(kat_path, dst, corrupt_index=None):
    algorithm, out_bits, vectors = load_kat_file(kat_path)
    lines = ["# re-emitted from " + kat_path.name, f"[{'Outputlen' if algorithm >= 4 else 'L'} = {out_bits}]", ""]
    for i, (msg, md) in enumerate(vectors):
        hexmd = md.hex()
        if i == corrupt_index:
            hexmd = ("0" if hexmd[0] != "0" else "1") + hexmd[1:]
        lines += [f"Len = {8 * len(msg)}", f"Msg = {msg.hex() if msg else '00'}", f"MD = {hexmd}", ""]
    dst.write_text("\n".join(lines))
    return len(vectors)


def run(cli, *args):
    return subprocess.run([str(cli), *args], capture_output=True, text=True, timeout=600)


def test_usage_and_io_errors(cli, tmp_path):
    """Exit codes of proj/tools/sha3cli/main.cpp:21-24 -- no GPU needed."""
    assert run(cli).returncode == 2
    assert run(cli, "bench", "--repeats", "2").returncode == 2           # < 3 repeats (runner.cpp:33-35)
    assert run(cli, "bench", "--algo", "md5").returncode == 2
    assert run(cli, "vectors", "--file", str(tmp_path / "missing.rsp"), "--algo", "sha3-256").returncode == 3
    odd = tmp_path / "data.rsp"
    odd.write_text("Len = 8\nMsg = 00\nMD = 00\n")
    assert run(cli, "vectors", "--file", str(odd)).returncode == 2        # cannot infer the algorithm
    bad = tmp_path / "SHA3_256bad.rsp"
    bad.write_text("Len = 12\nMsg = 0000\nMD = 00\n")
    r = run(cli, "vectors", "--file", str(bad))
    assert r.returncode == 3 and "byte-aligned" in r.stderr
    bad.write_text("Len = 8\nMD = 00\n")
    assert run(cli, "vectors", "--file", str(bad)).returncode == 3        # MD without Msg


MALFORMED = {
    # name -> (text, line both parsers must name)
    "len_not_aligned": ("Len = 12\nMsg = 0000\nMD = 00\n", 1),
    "digest_before_msg": ("# c\nLen = 8\nMD = 00\n", 3),
    "msg_without_len": ("\nMsg = 00\n", 2),
    "second_len": ("Len = 8\nMsg = 00\nLen = 8\n", 3),
    "unknown_key": ("Len = 8\nMsg = 00\nDigest = 00\n", 3),
    "no_equals": ("Len = 8\nMsg 00\n", 2),
    "odd_hex": ("Len = 8\nMsg = 000\nMD = 00\n", 2),
    "bad_hex": ("Len = 8\nMsg = 0g\nMD = 00\n", 2),
    "short_msg": ("Len = 24\nMsg = 0000\nMD = 00\n", 2),
    "empty_digest": ("Len = 8\nMsg = 00\nMD =\n", 3),
    "truncated": ("Len = 8\nMsg = 00\nMD = 00\nLen = 8\nMsg = 11\n", 5),
    "bad_outputlen": ("[Outputlen = x]\nLen = 8\nMsg = 00\nMD = 00\n", 1),
    "bad_len": ("Len = eight\n", 1),
}

WELL_FORMED = {
    "crlf_and_spaces": "[L = 256]\r\n\r\n  Len   =  16 \r\nMsg=ABcd\r\n\tMD = 00ff\r\n",
    "empty_message_placeholder": "Len = 0\nMsg = 00\nMD = a7\n",
    "msg_longer_than_len": "Len = 8\nMsg = 112233\nOutput = 0102\n",
    "msg_given_twice": "Len = 8\nMsg = 11\nMsg = 22\nMD = 0102\n",
    "other_headers": "[Foo]\n[Bar = 1]\n[Outputlen = 24]\nLen = 8\nMsg = 11\nOutput = 010203\n",
    "no_vectors": "# nothing\n\n",
}


def test_rsp_reader_matches_the_reference_parser(tmp_path):
    """Parser parity (f-2): paper_1902_05320_b200/host/rsp_reader.cpp against the reference's
    own parse_vector_file (vectors.cpp:42-125, compiled unmodified into oracle/_ref/rsp_parity)
    -- same vectors from well-formed files, same line named for malformed ones."""
    tool = ROOT / "oracle" / "_ref" / "rsp_parity"
    if not tool.exists():
        pytest.skip("oracle/_ref/rsp_parity not built (needs /root/reference)")
    files, expect = [], []
    for kat in sorted(GOLDEN.glob("*.kat")):
        dst = tmp_path / (kat.stem + ".rsp")
        n = write_rsp(kat, dst)
        files.append(dst)
        expect.append(f"same {n}")
    for name, text in WELL_FORMED.items():
        dst = tmp_path / (name + ".rsp")
        dst.write_bytes(text.encode())
        files.append(dst)
        expect.append("same")
    for name, (text, line) in MALFORMED.items():
        dst = tmp_path / (name + ".rsp")
        dst.write_bytes(text.encode())
        files.append(dst)
        expect.append(f"reject {line}")
    r = subprocess.run([str(tool), *map(str, files)], capture_output=True, text=True, timeout=120)
    rows = r.stdout.strip().splitlines()
    assert len(rows) == len(files), r.stdout + r.stderr
    for f, want, row in zip(files, expect, rows):
        assert row.startswith(f"{f} {want}"), row
    assert r.returncode == 0


def test_cli_names_the_line_of_a_malformed_file(cli, tmp_path):
    for name, (text, line) in MALFORMED.items():
        bad = tmp_path / ("sha3_256_" + name + ".rsp")
        bad.write_bytes(text.encode())
        r = run(cli, "vectors", "--file", str(bad))
        assert r.returncode == 3 and f"line {line}:" in r.stderr, (name, r.stderr)


@pytest.mark.gpu
@pytest.mark.parametrize("stem", ["SHA3_224ShortMsg", "SHA3_256LongMsg", "SHA3_384ShortMsg", "SHA3_512LongMsg",
                                  "SHAKE128ShortMsg", "SHAKE256LongMsg"])
def test_vectors_subcommand(cli, tmp_path, stem):
    rsp = tmp_path / (stem + ".rsp")
    n = write_rsp(GOLDEN / (stem + ".kat"), rsp)
    r = run(cli, "vectors", "--file", str(rsp))
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"{n}/{n} vectors passed" in r.stdout and "cuda" in r.stdout


@pytest.mark.gpu
def test_vectors_subcommand_reports_a_corrupted_digest(cli, tmp_path):
    """Fault injection as in proj/tests/acceptance.cpp:465-488: one flipped hex digit."""
    rsp = tmp_path / "SHA3_256ShortMsg.rsp"
    n = write_rsp(GOLDEN / "SHA3_256ShortMsg.kat", rsp, corrupt_index=17)
    r = run(cli, "vectors", "--file", str(rsp))
    assert r.returncode == 1
    assert "FAIL line" in r.stdout and f"{n - 1}/{n} vectors passed" in r.stdout


@pytest.mark.gpu
def test_bench_subcommand_csv(cli, tmp_path):
    """Same CSV columns as report.cpp:15-16, backend column `cuda`, Table-3 style sweep."""
    out = tmp_path / "bench.csv"
    r = run(cli, "bench", "--algo", "sha3-256", "--message-size", "10", "--sizes", "1202,37202,1190402",
            "--repeats", "3", "--csv", str(out))
    assert r.returncode == 0, r.stdout + r.stderr
    rows = list(csv.DictReader(out.open()))
    assert list(rows[0].keys()) == ["total_bytes", "message_size", "message_count", "backend",
                                    "time_seconds", "throughput_bps", "repeats"]
    assert [int(x["message_count"]) for x in rows] == [120, 3720, 119040]
    assert [int(x["total_bytes"]) for x in rows] == [1200, 37200, 1190400]   # hashed bytes (runner.cpp:42-43)
    for x in rows:
        assert x["backend"] == "cuda" and int(x["repeats"]) >= 3
        assert abs(float(x["throughput_bps"]) * float(x["time_seconds"]) - int(x["total_bytes"])) < 1.0
    assert "throughput_Bps" in r.stdout


@pytest.mark.gpu
def test_bench_subcommand_packed_layout(cli, tmp_path):
    """--layout packed: the same sweep on pinned packed buffers through b200sha3_hash_fixed."""
    out = tmp_path / "bench.csv"
    r = run(cli, "bench", "--algo", "shake128", "--bits", "1024", "--message-size", "64", "--sizes",
            "6400,67108864", "--layout", "packed", "--csv", str(out))
    assert r.returncode == 0, r.stdout + r.stderr
    rows = list(csv.DictReader(out.open()))
    assert [int(x["message_count"]) for x in rows] == [100, 1 << 20]
    assert all(x["backend"] == "cuda-packed" and int(x["repeats"]) >= 3 for x in rows)
    # 2^20 x 64 B over PCIe and back: comfortably above 1 GB/s of hashed input
    assert float(rows[1]["throughput_bps"]) > 1e9


@pytest.mark.gpu
def test_elapsed_is_the_wall_time_of_the_call(cli):
    """BatchResult::elapsed (the bench's time_s) covers pack + copies + kernels + unpack; the
    kernel-only time is a separate, much smaller column."""
    r = run(cli, "bench", "--message-size", "64", "--sizes", "67108864")
    assert r.returncode == 0, r.stdout + r.stderr
    cols = r.stdout.strip().splitlines()[-1].split()
    time_s, kernels_s = float(cols[4]), float(cols[7])
    assert 0 < kernels_s < time_s


@pytest.mark.gpu
@pytest.mark.parametrize("algo,bits,size", [("sha3-256", 0, 0), ("sha3-512", 0, 5_000_001), ("shake128", 2048, 777),
                                            ("SHA3_224", 0, 4 << 20), ("shake-256", 0, 136)])
def test_hash_subcommand(cli, tmp_path, algo, bits, size):
    """`hash FILE` streams the file through the device-resident incremental hasher."""
    import hashlib
    import numpy as np
    data = np.random.default_rng(size).integers(0, 256, size, dtype=np.uint8).tobytes()
    f = tmp_path / "blob.bin"
    f.write_bytes(data)
    args = ["hash", "--algo", algo] + (["--bits", str(bits)] if bits else []) + [str(f)]
    r = run(cli, *args)
    assert r.returncode == 0, r.stdout + r.stderr
    name = algo.lower().replace("-", "_").replace("shake_", "shake")
    name = {"shake128": "shake_128", "shake256": "shake_256"}.get(name, name)
    h = hashlib.new(name, data)
    if name.startswith("shake"):
        want = h.hexdigest((bits or (256 if name == "shake_128" else 512)) // 8)
    else:
        want = h.hexdigest()
    assert r.stdout.strip() == want
    assert run(cli, "hash", "--algo", "sha3-256", "--bits", "256", str(f)).returncode == 2
    assert run(cli, "hash", str(tmp_path / "missing")).returncode == 3


@pytest.mark.gpu
def test_reference_parser_on_our_backend(tmp_path):
    """The reference's unmodified vectors.cpp (parser) + the drop-in hash_batch: every response
    file verifies through the GPU (oracle/_ref/ref_runner_on_b200 vectors ...)."""
    tool = ROOT / "oracle" / "_ref" / "ref_runner_on_b200"
    if not tool.exists():
        pytest.skip("oracle/_ref/ref_runner_on_b200 not built (needs /root/reference at build time)")
    files = []
    total = 0
    for kat in sorted(GOLDEN.glob("*.kat")):
        dst = tmp_path / (kat.stem + ".rsp")
        total += write_rsp(kat, dst)
        files.append(str(dst))
    r = subprocess.run([str(tool), "vectors", *files], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    seen = sum(int(row.rsplit(" ", 1)[1].split("/")[0]) for row in r.stdout.strip().splitlines())
    assert seen == total == 892


@pytest.mark.gpu
def test_bench_packed_layout_on_few_long_messages(cli):
    """256 x 1 MiB from pinned memory: the piece pipeline of the fixed-length host entry, with its
    per-piece kernel timing (cfg->device_ms) -- kernel time is reported and is less than the call."""
    r = run(cli, "bench", "--message-size", "1048576", "--sizes", "268435456", "--layout", "packed")
    assert r.returncode == 0, r.stdout + r.stderr
    cols = r.stdout.strip().splitlines()[-1].split()
    assert int(cols[2]) == 256 and cols[3] == "cuda-packed"
    time_s, kernels_s = float(cols[4]), float(cols[7])
    assert 0.010 < kernels_s < time_s < 0.060          # ~16 ms of hashing inside a ~17-20 ms call
