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
