"""Deterministic test batches shared by the fixture generator and the tests."""
import json
import pathlib

GOLDEN = pathlib.Path(__file__).resolve().parent / "golden"


def materialize(oracle, kind, seed, count, max_len):
    """-> (messages, workload_total_bytes or None).

    kind "rng":      random_batch of proj/tests/test_batch.cpp:15-22 -- one
                     below(max_len+1) draw, then one draw per byte.
    kind "workload": `count` messages of `max_len` bytes from the head of the
                     reference's generate_workload stream (workload.cpp:16-47).
    """
    if kind == "rng":
        rng = oracle.test_rng(seed)
        return [rng.random_bytes(rng.below(max_len + 1)) for _ in range(count)], None
    size = max_len
    total = (1 << 26) if (size == 64 and count == 1 << 14) else count * size + (2 if size == 10 else 0)
    blob = oracle.generate_workload(total, size, seed=seed)[:count * size].tobytes()
    return [blob[i * size:(i + 1) * size] for i in range(count)], total


def ref_batch_cases():
    return json.loads((GOLDEN / "ref_batches.json").read_text())["cases"]
