"""Generate tests/golden/large_outputs.json: the UNMODIFIED reference's
results (oracle/_ref/libjsontape_ref.so) on the BASELINE.json configs at full
size, and on seeded single-error variants of the 1 GiB C4 document with the
error past byte 2^30.  Run here, where /root/reference (and so oracle/_ref)
exists; the GPU box regenerates the documents with tools/jtgen.c and compares
digests (tests/test_gpu_large.py).  About 5 minutes on 8 cores.

Each clean row: input sha256 (pins the generator), code, offset, S, T, string
bytes, and sha256 of index / tape / strings.  C3 (NDJSON): every record parsed
alone with jt_parse (the C3 semantics) and digested by
tests.large_cases.record_digest.  Error variants: the patch (position, bytes)
chosen from the reference's own index of the clean C4 document, then the
reference's code, offset and (unless UTF-8) index sha of the patched one.
"""
import ctypes as C
import hashlib
import json
import os
import random
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import ERROR_NAMES, Reference, _doc_words  # noqa: E402
from tests.large_cases import CLEAN, FIXTURE, RECORDS, document, mutate, record_digest, sha  # noqa: E402
from tools.gen import SEEDS, SIZES  # noqa: E402

ERR_FROM = 1 << 30


def clean_row(ref, name, cfg, size):
    d = document(cfg, size)
    t0 = time.time()
    r = ref.parse(d)
    row = {"name": name, "config": cfg, "size": size or SIZES[cfg], "seed": SEEDS[cfg], "bytes": len(d),
           "input_sha": sha(d), "code": ERROR_NAMES[r.code], "offset": r.offset,
           "S": len(r.index) // 4, "index_sha": sha(r.index)}
    if r.code == 0:
        row.update(T=len(r.tape) // 8, string_bytes=len(r.strings), tape_sha=sha(r.tape),
                   strings_sha=sha(r.strings))
    print(name, row["code"], len(d), "%.1fs" % (time.time() - t0), flush=True)
    return row, r


def records_row(ref):
    name, cfg, size = RECORDS
    d = document(cfg, size)
    recs = d.split(b"\n")
    if d.endswith(b"\n"):
        recs = recs[:-1]
    L = ref.lib
    codes = np.zeros(len(recs), np.int32)
    offs = np.zeros(len(recs), np.int64)
    tapes, strs = [], []
    t0 = time.time()
    for k, rec in enumerate(recs):
        doc = C.c_void_p()
        off = C.c_longlong(-7)
        code = L.jt_parse(ref.p, rec, len(rec), C.byref(doc), C.byref(off))
        codes[k] = code
        offs[k] = off.value
        if code == 0:
            tp, st = _doc_words(doc.value)
            tapes.append(tp)
            strs.append(st)
            L.jt_document_free(doc)
    row = {"name": name, "config": cfg, "size": size or SIZES[cfg], "seed": SEEDS[cfg], "bytes": len(d),
           "input_sha": sha(d)}
    row.update(record_digest(codes, offs, b"".join(tapes), b"".join(strs)))
    row["failed_codes"] = {ERROR_NAMES[c]: int((codes == c).sum()) for c in np.unique(codes) if c}
    print(name, row["records"], "records", "%.1fs" % (time.time() - t0), flush=True)
    return row


def pick(idx, data, lo, pred, rng):
    """A seeded index entry at or past byte `lo` whose byte satisfies pred."""
    cand = np.nonzero(idx >= lo)[0]
    rng.shuffle(cand_list := list(cand))
    for k in cand_list:
        if pred(int(k)):
            return int(k)
    raise RuntimeError("no candidate")


def error_variants(ref, d, r):
    """Single-error variants of the clean C4 document, errors past 2^30."""
    idx = np.frombuffer(r.index, dtype=np.uint32).astype(np.int64)
    nxt = lambda k: int(idx[k + 1]) if k + 1 < len(idx) else len(d)  # noqa: E731
    byte = lambda k: d[int(idx[k])]  # noqa: E731
    rng = random.Random(1073741824)
    plans = []

    def string_content(k):  # an opening quote with >= 4 content bytes before the next token
        return byte(k) == ord('"') and nxt(k) - int(idx[k]) >= 6 and d[int(idx[k]) + 1] != ord("\\")

    def number(k):
        return chr(byte(k)) in "123456789" and nxt(k) - int(idx[k]) >= 3 and \
            chr(d[int(idx[k]) + 1]) in "0123456789"
    # 1 invalid UTF-8 inside a string
    k = pick(idx, d, ERR_FROM, string_content, rng)
    plans.append(("invalid UTF-8 (0xFF) in a string", [int(idx[k]) + 2, "ff"]))
    # 2 overlong UTF-8 (C0 AF = '/')
    k = pick(idx, d, ERR_FROM, string_content, rng)
    plans.append(("overlong UTF-8 (C0 AF) in a string", [int(idx[k]) + 1, "c0af"]))
    # 3 unbalanced / mismatched bracket: a closer flipped
    k = pick(idx, d, ERR_FROM, lambda k: byte(k) in b"]}", rng)
    plans.append(("mismatched closing bracket", [int(idx[k]), "7d" if byte(k) == ord("]") else "5d"]))
    # 3b an extra opener: a ',' turned into '['
    k = pick(idx, d, ERR_FROM, lambda k: byte(k) == ord(","), rng)
    plans.append(("unbalanced bracket (',' -> '[')", [int(idx[k]), "5b"]))
    # 4 raw control char in a string
    k = pick(idx, d, ERR_FROM, string_content, rng)
    plans.append(("raw control char (0x1f) in a string", [int(idx[k]) + 3, "1f"]))
    k = pick(idx, d, ERR_FROM, string_content, rng)
    plans.append(("raw newline in a string", [int(idx[k]) + 1, "0a"]))
    # 5 bad number: leading zero, and a letter inside the digits
    k = pick(idx, d, ERR_FROM, number, rng)
    plans.append(("bad number (leading zero)", [int(idx[k]), "30"]))
    k = pick(idx, d, ERR_FROM, number, rng)
    plans.append(("bad number (letter in digits)", [int(idx[k]) + 1, "78"]))
    rows = []
    for what, patch in plans:
        m = mutate(d, patch)
        t0 = time.time()
        rr = ref.parse(m)
        row = {"name": "C4 " + what, "config": 4, "patch": patch, "code": ERROR_NAMES[rr.code],
               "offset": rr.offset}
        if rr.code != 1:
            row["index_sha"] = sha(rr.index)
            row["S"] = len(rr.index) // 4
        assert rr.code != 0, what
        print(row["name"], row["code"], row["offset"], "%.1fs" % (time.time() - t0), flush=True)
        rows.append(row)
    return rows


def main():
    ref = Reference()
    out = {"generated_by": "tests/golden/make_golden_large.py (oracle/_ref = unmodified reference)",
           "clean": [], "errors": [], "records": None}
    for name, cfg, size in CLEAN:
        row, r = clean_row(ref, name, cfg, size)
        out["clean"].append(row)
        if cfg == 4:
            out["errors"] = error_variants(ref, document(cfg, size), r)
        del r
    out["records"] = records_row(ref)
    with open(FIXTURE, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", FIXTURE)


if __name__ == "__main__":
    main()
