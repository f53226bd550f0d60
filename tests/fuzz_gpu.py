"""Long-running differential fuzz of the GPU paths against the oracle.

python tests/fuzz_gpu.py --seconds 600 [--seed N]   (test infrastructure: it runs the oracle)

Each round draws a document (generated configs C0..C4 at random sizes, random
JSON, byte soups, and seeded mutations of all of them) and checks, against
the oracle (tests/ pin the oracle to the reference):
  jt_parse (in-memory and, >= 8 MiB, the streamed path), emulated byte-range
  shards (2..6), NDJSON records, jt_minify, jt_compute_stats, jt_stage1 (the
  k_index path) and the device distinct_values query (against the host walk).
Prints one line per failure (document saved under gpurun_out/fuzz_fail_*.bin)
and a summary; exit status 1 if anything failed.
"""
from __future__ import annotations

import argparse
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle.pyoracle import Oracle  # noqa: E402
from paper_1902_08318_b200 import Parser  # noqa: E402
from tests.test_gpu_parity import _mutate, _rand_json  # noqa: E402
from tests.vectors import SOUP_POOL  # noqa: E402
from tools.gen import generate  # noqa: E402


def draw(rng: random.Random) -> bytes:
    k = rng.randrange(12)
    if k >= 10:  # strings of escape sequences at every block alignment (some with failing escapes)
        from tests.test_kernels_cpu import _escape_soup
        parts = [_escape_soup(rng, rng.random() < 0.15) for _ in range(rng.randrange(1, 60))]
        return b"[" + b",".join(parts) + b"]"
    if k < 4:
        cfg = rng.choice([0, 1, 2, 4])
        size = rng.choice([1 << 12, 1 << 14, 100000, 1 << 18, 1 << 20, 3 << 20])
        d = generate(cfg, size, seed=rng.randrange(1 << 30))
    elif k < 7:
        d = _rand_json(rng).encode()
        if rng.random() < 0.3:  # pretty-print-ish whitespace
            d = d.replace(b",", b",\n  ").replace(b":", b": ")
    elif k < 8:
        d = bytes(rng.choice(SOUP_POOL) for _ in range(rng.randrange(0, 3000)))
    else:
        d = b"[" + b",".join(_rand_json(rng).encode() for _ in range(rng.randrange(1, 400))) + b"]"
    if rng.random() < 0.4:
        for _ in range(rng.randrange(1, 4)):
            d = _mutate(rng, d)
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=1902)
    args = ap.parse_args()
    rng = random.Random(args.seed)
    o, p = Oracle(), Parser()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    t0 = time.time()
    n = fails = 0
    counts = {"parse": 0, "shards": 0, "records": 0, "minify": 0, "stats": 0, "streamed": 0, "stage1": 0,
              "distinct": 0}

    def fail(what, d, detail):
        nonlocal fails
        fails += 1
        path = os.path.join(ROOT, "gpurun_out", f"fuzz_fail_{fails}.bin")
        with open(path, "wb") as f:
            f.write(d)
        print(f"FAIL {what}: {detail} ({len(d)} bytes, saved {path})", flush=True)

    while time.time() - t0 < args.seconds:
        d = draw(rng)
        n += 1
        r = o.parse(d)
        g = p.parse(d)
        counts["parse"] += 1
        if (g.name, g.offset) != (r.name, r.offset):
            fail("parse", d, (g.name, g.offset, r.name, r.offset))
            continue
        if r.code == 0 and (not np.array_equal(g.document.tape, r.tape_array()) or g.document.strings != r.strings):
            fail("parse tape", d, "tape/strings differ")
            continue
        if r.code == 0 and rng.random() < 0.3:  # device distinct_values on this parse
            import re
            keys = [m.group(1) for m in re.finditer(rb'"([^"\\\x00]{1,16})"\s*:', d[:1 << 16])][:8]
            for path in [k for k in keys[:3]] + [a + b"." + b for a, b in zip(keys[:3], keys[1:4])]:
                counts["distinct"] += 1
                if p.distinct(path) != g.document.distinct(path):
                    fail("distinct", d, path)
                    break
        if rng.random() < 0.3:  # jt_stage1 alone (k_index)
            s1g, s1o = p.stage1(d), o.stage1(d)
            counts["stage1"] += 1
            if (s1g.name, s1g.offset) != (s1o.name, s1o.offset) or (
                    s1o.code == 0 and not np.array_equal(p.index(), s1o.index_list())):
                fail("stage1", d, (s1g.name, s1g.offset, s1o.name, s1o.offset))
        if rng.random() < 0.1 and len(d) > 0:  # a big streamed variant: the doc in a 9+ MiB array
            reps = max(1, (9 << 20) // max(1, len(d)) + 1)
            if r.code == 0 and reps * len(d) < (40 << 20):
                big = b"[" + b",".join([d] * reps) + b"]"
                rb = o.parse(big)
                for mode, q in (("streamed", p),):
                    gb = q.parse(big)
                    counts["streamed"] += 1
                    if (gb.name, gb.offset) != (rb.name, rb.offset) or (
                            rb.code == 0 and (not np.array_equal(gb.document.tape, rb.tape_array())
                                              or gb.document.strings != rb.strings)):
                        fail(mode, big, (gb.name, gb.offset, rb.name, rb.offset))
        tiles = (len(d) + 16383) // 16384
        if tiles >= 2 and rng.random() < 0.5:
            from paper_1902_08318_b200.shard import LocalShards
            G = rng.randrange(2, min(6, tiles) + 1)
            ls = LocalShards(d, G)
            try:
                name, off = ls.run()
                counts["shards"] += 1
                if (name, off) != (r.name, r.offset):
                    fail(f"shards G={G}", d, (name, off, r.name, r.offset))
                elif r.code == 0:
                    tape, strings = ls.assemble()
                    if not np.array_equal(tape, r.tape_array()) or strings != r.strings:
                        fail(f"shards G={G} tape", d, "tape/strings differ")
            finally:
                ls.close()
        if rng.random() < 0.3:
            lines = [draw(rng).replace(b"\n", b" ") for _ in range(rng.randrange(1, 30))]
            buf = b"\n".join(lines) + (b"\n" if rng.random() < 0.5 else b"")
            import torch
            host = torch.frombuffer(bytearray(buf), dtype=torch.uint8) if buf else torch.zeros(1, dtype=torch.uint8)
            p.copy_in(host.data_ptr(), len(buf))
            got = p.parse_records(len(buf))
            recs = buf.split(b"\n")
            if buf.endswith(b"\n"):
                recs = recs[:-1]
            if not buf:
                recs = []
            counts["records"] += 1
            if len(got) != len(recs):
                fail("records count", buf, (len(got), len(recs)))
            else:
                for k, (rec, gr) in enumerate(zip(recs, got)):
                    orr = o.parse(rec)
                    if (gr[0], gr[1]) != (orr.name, orr.offset) or (
                            orr.code == 0 and (not np.array_equal(gr[2], orr.tape_array()) or gr[3] != orr.strings)):
                        fail(f"record {k}", buf, (gr[0], gr[1], orr.name, orr.offset))
                        break
        if rng.random() < 0.2:
            counts["minify"] += 1
            if p.minify(d) != o.minify(d):
                fail("minify", d, "differs")
        if rng.random() < 0.2:
            counts["stats"] += 1
            if p.stats(d) != o.stats(d):
                fail("stats", d, "differs")
    print(f"fuzz: {n} documents in {time.time() - t0:.0f} s, {counts}, failures {fails}", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
