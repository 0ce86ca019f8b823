"""The multi-rank CUDA path of bench.py under a real process group: one
process per rank launched by torch.distributed.run exactly as the driver launches the
scaling run, each rank hashing its contiguous message range with the CUDA kernels -- the
fan-out of proj/core/src/batch.cpp:94-127 one level up.

On a one-GPU box the ranks share device 0 (`--share-gpu`: gloo process group, the same
shard / barrier / all-reduce code path, numbers not benchmark values); with two or more
devices visible the NCCL branch runs as the driver runs it.  Either way the sharded result
must equal the single-process one: same digest checksum, and kernel launches that sum over
ranks."""
import json
import os
import pathlib
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = pathlib.Path(__file__).resolve().parent.parent
LOG2 = 22
STEPS, WARMUP = 2, 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(ranks, *extra):
    common = ["--gpus", str(ranks), "--steps", str(STEPS), "--warmup", str(WARMUP), "--log2-messages", str(LOG2),
              "--no-cpu-baseline", "--no-configs", "--no-dropin", "--no-probe", *extra]
    if ranks == 1:
        cmd = [sys.executable, "bench.py", *common]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", *common]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(ROOT), env=env)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout          # rank 0 alone prints
    return json.loads(lines[0])


@pytest.fixture(scope="module")
def single():
    return _bench(1)


def _check_sharded(line, single, ranks):
    assert line["n_gpus"] == ranks and line["config"]["messages_total"] == 1 << LOG2
    assert line["config"]["messages_per_gpu"] == (1 << LOG2) // ranks
    assert line["digest_checksum"] == single["digest_checksum"]      # same digests, however sharded
    assert single["gpu_launches"] == STEPS                           # one kernel per step ...
    assert line["gpu_launches"] == STEPS * ranks                     # ... per rank, summed over ranks
    assert line["value"] > 0 and line["scaling"] == "strong"
    e2e = line["e2e"]
    assert e2e["digests_match_device_path"] is True
    assert e2e["h2d_bytes_per_step"] == (1 << LOG2) * 64 and e2e["d2h_bytes_per_step"] == (1 << LOG2) * 32


@pytest.mark.parametrize("ranks", [2, 4])
def test_ranks_sharing_one_gpu_match_the_single_rank_run(single, ranks):
    line = _bench(ranks, "--share-gpu", "--gather-digests")
    assert "validation_only" in line
    _check_sharded(line, single, ranks)
    # the optional gather after the hot path: every rank holds all digests, in message order
    assert line["digest_gather"]["checksum_matches"] is True
    assert line["digest_gather"]["bytes_per_rank"] == (1 << LOG2) * 32


def test_nccl_branch_when_two_devices_are_visible(single):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one CUDA device visible: the NCCL branch needs two (the gloo/shared-GPU test above "
                    "covers the same shard, barrier and reduction code)")
    line = _bench(2, "--gather-digests")
    assert "validation_only" not in line
    _check_sharded(line, single, 2)
    assert line["digest_gather"]["checksum_matches"] is True and line["digest_gather"]["backend"] == "nccl"


@pytest.mark.parametrize("ranks", [2, 3])
def test_variable_length_batch_sharded_by_block_count(ranks):
    """SURVEY.md 8(e), variable-length half: contiguous ranges balanced by cumulative block count,
    each rank hashing its range with the CUDA path under a process group; the concatenation is
    the unsharded result and the ranges carry near-equal work."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "tests" / "integration" / "multirank_ragged.py"), "30000"]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=str(ROOT), env=env)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["ranks"] == ranks and rec["sharded_equals_unsharded"] is True and rec["oracle_sample_ok"] is True
    assert sum(c for _, c in rec["ranges"]) == 30000
    work = rec["blocks_per_rank"]
    assert max(work) - min(work) <= 2 * (200000 // 136 + 1)      # within a heaviest message or two
