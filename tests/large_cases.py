"""Full-size parity cases: the BASELINE.json configs at the sizes the bench
runs them (C0 1 MiB, C1 64 MiB, C2 256 MiB, C3 1 GiB NDJSON, C4 1 GiB), plus
seeded single-error variants of the C4 document with the error placed past
byte 2^30 (the C4 document is 1,073,786,410 bytes, so [2^30, len) is a 44 KB
window at its end: offsets that only a >1 GiB document reaches).

The expected results come from the UNMODIFIED reference (oracle/_ref, built
from /root/reference) and are committed in tests/golden/large_outputs.json by
tests/golden/make_golden_large.py; the GPU tests regenerate the documents with
tools/jtgen.c on the box and compare sha256 digests.  An error variant is the
clean document with one recorded byte patch (position + bytes) chosen from the
reference's own structural index of the clean document, so the box applies
exactly the same mutation without re-deriving it.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURE = os.path.join(HERE, "golden", "large_outputs.json")

# (name, config, size) - size None = tools.gen.SIZES[config]
CLEAN = [("C0", 0, None), ("C1", 1, None), ("C2", 2, None), ("C4", 4, None)]
RECORDS = ("C3", 3, None)


def sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def load_fixture() -> dict:
    with open(FIXTURE) as f:
        return json.load(f)


_DOCS: dict = {}


def document(config: int, size=None) -> bytes:
    """The seeded config document (cached: C4 takes ~14 s to generate)."""
    key = (config, size)
    if key not in _DOCS:
        from tools.gen import generate
        _DOCS[key] = generate(config, size)
    return _DOCS[key]


def mutate(doc: bytes, patch) -> bytes:
    """Apply a recorded [position, hex bytes] patch (same length: no shift)."""
    pos, hexb = patch
    b = bytes.fromhex(hexb)
    out = bytearray(doc)
    out[pos:pos + len(b)] = b
    return bytes(out)


def record_digest(codes: np.ndarray, offsets: np.ndarray, tape_words_ok: bytes, strings_ok: bytes) -> dict:
    """Per-record results of an NDJSON buffer, digested: code and offset of
    every record (jt_parse(record) semantics), and the concatenation over the
    OK records, in order, of their tape words and of their string buffers."""
    return {
        "records": int(len(codes)),
        "ok": int((codes == 0).sum()),
        "codes_sha": sha(np.ascontiguousarray(codes, dtype=np.int32).tobytes()),
        "offsets_sha": sha(np.ascontiguousarray(offsets, dtype=np.int64).tobytes()),
        "tape_sha": sha(tape_words_ok),
        "strings_sha": sha(strings_ok),
    }


def gather_ranges(buf: np.ndarray, begin: np.ndarray, count: np.ndarray) -> np.ndarray:
    """Concatenate buf[begin[k]:begin[k]+count[k]] for all k (vectorised)."""
    count = count.astype(np.int64)
    total = int(count.sum())
    if total == 0:
        return buf[:0]
    starts = np.repeat(begin.astype(np.int64) - np.concatenate(([0], np.cumsum(count)[:-1])), count)
    return buf[starts + np.arange(total, dtype=np.int64)]
