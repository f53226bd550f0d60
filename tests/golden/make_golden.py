"""Generate tests/golden/reference_outputs.jsonl from the UNMODIFIED reference
(oracle/_ref/libjsontape_ref.so, built from /root/reference by
oracle/build_ref.sh).  Run here, where /root/reference exists; the fixture is
committed so tests on the GPU box need no reference sources.

Each row: the input (hex, or a jtgen recipe [config, size, seed, err]), the
reference's code name and offset, and sha256 of its index, tape and string
buffer (tape/strings only on OK)."""
import hashlib
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import ERROR_NAMES, Reference  # noqa: E402
from tests.test_gpu_parity import _mutate, _rand_json  # noqa: E402
from tests.vectors import KAT, SOUP_POOL  # noqa: E402
from tools.gen import generate  # noqa: E402


def row(ref, data, recipe=None):
    r = ref.parse(data)
    out = {"code": ERROR_NAMES[r.code], "offset": r.offset}
    if recipe is None:
        out["input"] = data.hex()
    else:
        out["gen"] = recipe
    if r.code != 1 and r.index is not None:
        out["index_sha"] = hashlib.sha256(r.index).hexdigest()
    if r.code == 0:
        out["tape_sha"] = hashlib.sha256(r.tape).hexdigest()
        out["strings_sha"] = hashlib.sha256(r.strings).hexdigest()
    return out


def main():
    ref = Reference()
    rows = []
    for data, _, _ in KAT:
        rows.append(row(ref, data))
    rng = random.Random(1902)
    for _ in range(150):
        rows.append(row(ref, bytes(rng.choice(SOUP_POOL) for _ in range(rng.randrange(0, 300)))))
    for _ in range(150):
        d = _rand_json(rng).encode()
        rows.append(row(ref, d))
        rows.append(row(ref, _mutate(rng, d)))
    for cfg, size in [(0, 1 << 16), (1, 1 << 17), (2, 1 << 17), (4, 1 << 17)]:
        rows.append(row(ref, generate(cfg, size, seed=7), [cfg, size, 7, 0]))
    for seed in range(1, 41):
        err = 1 + seed % 5
        rows.append(row(ref, generate(4, 1 << 13, seed=seed, err=err), [4, 1 << 13, seed, err]))
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_outputs.jsonl")
    with open(out, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
    print("wrote", out, len(rows))


if __name__ == "__main__":
    main()
