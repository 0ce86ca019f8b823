"""bench.py on a GPU box, reduced sizes: the JSON line carries every key the contract and
VERDICT round 1 ask for -- roofline with the executed-instruction view, e2e with its copy
sizes, the cfg1..cfg4 points (+ the few-long-messages point), both CPU baseline builds."""
import json
import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parent.parent


def test_bench_line_shape_at_reduced_size():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--log2-messages", "22",
                          "--quick-configs", "--no-dropin", "--cpu-log2-messages", "16"],
                         capture_output=True, text=True, timeout=900, cwd=str(ROOT), env=env)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["metric"] == "SHA3-256 hashes/s on 64-B msg batches" and line["unit"] == "hashes/s"
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["gpu_launches"] == 3 and line["value"] > 1e9
    roof = line["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic", "instr_per_hash_contract",
                "instr_executed_per_hash", "frac_executed", "algorithmic_bytes_per_launch"):
        assert key in roof, key
    assert roof["instr_per_hash_contract"] == 4320
    if roof["instr_executed_per_hash"] is not None:        # profiles/sass_census.json present
        assert 4000 < roof["instr_executed_per_hash"] < 4320
        assert abs(roof["frac_executed"] * 4320 - roof["frac"] * roof["instr_executed_per_hash"]) < 1e-6 * 4320
    e2e = line["e2e"]
    assert e2e["h2d_bytes_per_step"] == (1 << 22) * 64 and e2e["d2h_bytes_per_step"] == (1 << 22) * 32
    assert e2e["digests_match_device_path"] is True and 0 < e2e["value"] < line["value"]
    # the link's ceiling for the call's shape, measured in the same run: both plain copies at once
    duplex = e2e["pcie"]["duplex_plain_copies"]
    assert duplex["ms"] > 0 and duplex["h2d_gb_per_s"] > 0 and e2e["pcie"]["e2e_step_over_duplex_copies"] > 0
    names = [c["config"] for c in line["configs"]]
    assert [n.split(":")[0] for n in names] == ["cfg1", "cfg2", "cfg2", "cfg2", "cfg3", "cfg3", "cfg4",
                                                "few long messages"]
    for c in line["configs"]:
        assert c["ms"] > 0 and c["hashes_per_s"] > 0 and 0 < c["int_roofline_frac"] < 1.2 and c["kernel"]
    assert line["configs"][-1]["kernel"] == "hash_warp_kernel"
    assert line["configs"][-1]["ms"] < line["configs"][-1]["ms_one_message_per_thread"]
    base = line["cpu_baseline"]
    assert base["kind"] in ("reference", "port") and base["cores"] >= 1 and base["value"] > 0
    if base["kind"] == "reference":
        assert set(base["builds_hashes_per_s"]) <= {"as_shipped", "hash_into"} and base["build"] in base["builds_hashes_per_s"]
    assert set(line["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    # build provenance of the library that ran
    assert "sm_100a" in line["library"]["version"] and line["library"]["path"].endswith("libb200sha3.so")
