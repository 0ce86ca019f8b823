#!/usr/bin/env python3
"""Golden outputs of the COMPILED REFERENCE for batches its .rsp files do not
cover (multi-block squeeze, odd XOF bit lengths, variable-length batches,
the cfg1 workload stream).  Run in the build container:

    make -C oracle && python tests/golden/make_ref_fixtures.py

Writes tests/golden/ref_batches.json.  Messages are not stored: they are
regenerated from the seed with the reference's test RNG (one splitmix64 draw
per byte, proj/tests/test_util.hpp:14-35) or its workload generator
(proj/tools/sha3cli/workload.cpp:16-47); per case the file keeps the SHA3-256
(hashlib) checksum of the concatenated reference digests plus the first and
last digest in clear.
"""
import hashlib
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent.parent
sys.path.insert(0, str(ROOT))

sys.path.insert(0, str(ROOT / "tests"))

from batches import materialize  # noqa: E402
from oracle.binding import Oracle, Reference, pack  # noqa: E402

CASES = [
    # (name, kind, algorithm, xof_bits, seed, count, max_len)
    ("test_batch_seed52_sha3_256", "rng", 1, 0, 52, 2000, 300),
    ("test_batch_seed53_order", "rng", 1, 0, 53, 500, 40),
    ("acceptance_seed_e9_sha3_512", "rng", 3, 0, 0xE9, 10000, 199),
    ("var_sha3_224", "rng", 0, 0, 1001, 3000, 700),
    ("var_sha3_384", "rng", 2, 0, 1002, 3000, 700),
    ("shake128_328bits", "rng", 4, 328, 1003, 2000, 400),
    ("shake128_4096bits", "rng", 4, 4096, 1004, 1500, 200),
    ("shake128_4099bits", "rng", 4, 4099, 1005, 1500, 200),
    ("shake256_512bits", "rng", 5, 512, 1006, 2000, 400),
    ("shake256_2048bits", "rng", 5, 2048, 1007, 1500, 200),
    ("shake256_1bit", "rng", 5, 1, 1008, 300, 50),
    ("shake256_12bits", "rng", 5, 12, 1009, 300, 50),
    ("long_sha3_256", "rng", 1, 0, 1010, 64, 20000),
    ("long_shake128", "rng", 4, 1344 * 3 + 8, 1011, 64, 20000),
    ("workload_cfg1_head_sha3_256", "workload", 1, 0, 1, 1 << 14, 64),
    ("workload_10byte_sha3_256", "workload", 1, 0, 1, 120, 10),
    ("workload_1k_sha3_512", "workload", 3, 0, 1, 4096, 1024),
    ("workload_64_shake256_4096", "workload", 5, 4096, 1, 4096, 64),
]


def main():
    oracle, ref = Oracle(), Reference()
    out = {"_generated_by": "tests/golden/make_ref_fixtures.py from oracle/_ref (compiled /root/reference)",
           "cases": []}
    for name, kind, algorithm, bits, seed, count, max_len in CASES:
        msgs, total = materialize(oracle, kind, seed, count, max_len)
        if kind == "workload":
            # the message bytes themselves must be the reference generator's
            assert (ref.generate_workload(total, max_len, seed=seed)[:count * max_len].tobytes()
                    == b"".join(msgs))
        data, offsets, lengths = pack(msgs)
        digests = ref.hash_batch(algorithm, data, offsets, lengths, xof_bits=bits, parallel=True)
        seq = ref.hash_batch(algorithm, data, offsets, lengths, xof_bits=bits, parallel=False)
        assert (digests == seq).all()
        out["cases"].append({
            "name": name, "kind": kind, "algorithm": algorithm, "xof_bits": bits, "seed": seed,
            "count": count, "max_len": max_len, "workload_total_bytes": total,
            "digest_bytes": int(digests.shape[1]),
            "checksum_sha3_256": hashlib.sha3_256(digests.tobytes()).hexdigest(),
            "first": digests[0].tobytes().hex(), "last": digests[-1].tobytes().hex(),
        })
        print(name, out["cases"][-1]["checksum_sha3_256"][:16])
    (pathlib.Path(__file__).parent / "ref_batches.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
