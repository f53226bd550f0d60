"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): every
kernel of the library on small inputs, each result checked against the
oracle so a silent corruption also fails.

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
    (see tools/sanitize.sh for the three tools and the logs kept in profiles/)

Paths: jt_parse single upload (< 8 MiB) and streamed (pieces, stage-2 token
ranges; pinned and pageable input), jt_stage1 (k_index) + jt_stage2, the
device-resident parse, NDJSON records, byte-range shards emulated on one GPU,
jt_minify, jt_compute_stats, device distinct_values.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from oracle.pyoracle import Oracle
    from paper_1902_08318_b200 import Parser
    from paper_1902_08318_b200.shard import LocalShards
    from tools.gen import generate

    small = os.environ.get("JT_SAN_SMALL", "0") == "1"
    o = Oracle()
    p = Parser()
    docs = [generate(c, 1 << 16, seed=5 + c) for c in (0, 1, 2, 4)]
    docs += [generate(4, 1 << 14, seed=9, err=k) for k in range(1, 6)]
    docs += [b'{"a": [1, 2.5e-3, "x\\u00e9\\ud83d\\ude00", true, null], "b": {}}', b"[1, 2", b'["\xff"]', b""]
    for d in docs:
        g, r = p.parse(d), o.parse(d)
        assert (g.name, g.offset) == (r.name, r.offset), (d[:40], g.name, r.name)
        if r.code == 0:
            assert np.array_equal(g.document.tape, r.tape_array()) and g.document.strings == r.strings
        g1 = p.stage1(d)
        assert g1.name == r.name or r.code != 1 or g1.name == "UTF8_ERROR"
        if g1.name == "OK":
            g2 = p.stage2()
            assert (g2.name, g2.offset) == (r.name, r.offset)
    print("single documents ok", flush=True)

    # streamed jt_parse (>= 8 MiB): pageable and pinned input
    big = generate(4 if small else 1, 9 << 20, seed=77)
    r = o.parse(big)
    g = p.parse(big)
    assert (g.name, g.offset) == (r.name, r.offset) and np.array_equal(g.document.tape, r.tape_array())
    assert g.document.strings == r.strings
    pin = torch.frombuffer(bytearray(big), dtype=torch.uint8).pin_memory()
    import ctypes as C
    doc = C.c_void_p()
    assert p._lib.jt_parse(p._h, C.c_char_p(pin.data_ptr()), len(big), C.byref(doc), None) == 0
    p._lib.jt_document_free(doc)
    print("streamed ok", flush=True)

    # device-resident parse, minify, stats, distinct
    d = docs[1]
    host = torch.frombuffer(bytearray(d), dtype=torch.uint8)
    p.copy_in(host.data_ptr(), len(d))
    assert p.parse_resident(len(d)).name == "OK"
    assert p.distinct(b"a") == p.download().distinct(b"a")
    assert p.minify(d) == o.minify(d)
    assert p.stats(d) == o.stats(d)
    print("resident / minify / stats / distinct ok", flush=True)

    # NDJSON records
    recs = generate(3, 1 << 16, seed=3) + b'{"a":[1,}\n"\\q"\n\n[1]'
    host = torch.frombuffer(bytearray(recs), dtype=torch.uint8)
    p.copy_in(host.data_ptr(), len(recs))
    got = p.parse_records(len(recs))
    lines = recs.split(b"\n")
    assert len(got) == len(lines)
    for line, gr in zip(lines, got):
        rr = o.parse(line)
        assert (gr[0], gr[1]) == (rr.name, rr.offset)
    print("records ok", flush=True)

    # byte-range shards (3, emulated on this GPU)
    d = generate(1, 3 << 16, seed=21)
    sh = LocalShards(d, 3)
    name, off = sh.run()
    r = o.parse(d)
    assert (name, off) == (r.name, r.offset)
    tape, strings = sh.assemble()
    assert np.array_equal(tape, r.tape_array()) and strings == r.strings
    sh.close()
    print("shards ok", flush=True)
    p.close()
    torch.cuda.synchronize()
    print("sanitize driver ok", flush=True)


if __name__ == "__main__":
    main()
