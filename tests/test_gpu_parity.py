"""GPU parity: the B200 kernels (through the C ABI) vs the CPU oracle.

Bit-exact: code, offset, structural index, tape words (incl. float64 bit
patterns) and string buffer.  Oracle = oracle/jt_oracle.c, itself pinned to
the reference (tests/test_oracle_*.py).
"""
import random

import numpy as np
import pytest

from tests.vectors import EXAMPLE_DOCUMENT, EXAMPLE_INTS, EXAMPLE_TAPE_WORDS, INDEX_KAT, KAT, SOUP_POOL

pytestmark = pytest.mark.gpu


def check_same(parser, oracle, data: bytes, where=""):
    g = parser.parse(data)
    o = oracle.parse(data)
    assert (g.name, g.offset) == (o.name, o.offset), (where, data[:200])
    if o.code == 0:
        d = g.document
        assert d is not None
        assert np.array_equal(d.tape, o.tape_array()), (where, data[:200])
        assert d.strings == o.strings, where
    if o.code != 1:  # stage-1 index refreshed unless UTF-8 failed
        assert np.array_equal(parser.index(), o.index_list()), (where, data[:200])
    return g


def test_kat_vectors(parser, oracle):
    for data, name, off in KAT:
        g = check_same(parser, oracle, data, "kat")
        assert g.name == name, data
        if off is not None:
            assert g.offset == off, data


def test_example_document_tape(parser):
    r = parser.parse(EXAMPLE_DOCUMENT)
    assert r.name == "OK"
    t = r.document.tape
    assert len(t) == 38
    for i, (tag, payload) in EXAMPLE_TAPE_WORDS.items():
        assert int(t[i]) >> 56 == ord(tag) and int(t[i]) & ((1 << 56) - 1) == payload
    for i, v in EXAMPLE_INTS:
        assert int(t[i]) >> 56 == ord("l")
        assert np.int64(t[i + 1].view(np.int64)) == v


def test_index_kat(parser):
    for data, expect in INDEX_KAT:
        r = parser.stage1(data)
        assert r.name == "OK"
        assert parser.index().tolist() == expect, data


def test_stage1_then_stage2(parser):
    src = b'{ "k" : [ 1 , 2 ] }'
    assert parser.stage1(src).name == "OK"
    assert parser.index().tolist() == [0, 2, 6, 8, 10, 12, 14, 16, 18]
    assert parser.stage2(want_document=False).name == "OK"
    a = parser.stage2()
    b = parser.parse(src)
    assert a.document == b.document


def test_soup_fuzz(parser, oracle):
    rng = random.Random(17)
    for it in range(3000):
        n = rng.randrange(0, 2000)
        data = bytes(rng.choice(SOUP_POOL) for _ in range(n))
        check_same(parser, oracle, data, f"soup {it}")


def _rand_json(rng, depth=0):
    k = rng.randrange(10 if depth < 6 else 6)
    if k == 0:
        return str(rng.randrange(-10**20, 10**20))
    if k == 1:
        return repr(rng.uniform(-1e10, 1e10)) if rng.random() < 0.5 else "%.17g" % (rng.random() * 10 ** rng.randrange(-300, 300))
    if k == 2:
        return rng.choice(["true", "false", "null"])
    if k in (3, 4, 5):
        chars = []
        for _ in range(rng.randrange(0, 40)):
            r = rng.random()
            if r < 0.1:
                chars.append(rng.choice(['\\"', "\\\\", "\\n", "\\t", "\\u00e9", "\\ud834\\udd1e", "\\/"]))
            elif r < 0.3:
                chars.append(rng.choice(["é", "€", "𝄞", "ж"]))
            else:
                chars.append(rng.choice("abcdefgh ,:[]{}"))
        return '"' + "".join(chars) + '"'
    if k in (6, 7):
        return "[" + ",".join(_rand_json(rng, depth + 1) for _ in range(rng.randrange(0, 6))) + "]"
    return "{" + ",".join('"k%d":%s' % (i, _rand_json(rng, depth + 1)) for i in range(rng.randrange(0, 6))) + "}"


def _mutate(rng, b: bytes) -> bytes:
    if not b:
        return b
    p = rng.randrange(len(b))
    op = rng.randrange(5)
    if op == 0:
        return b[:p] + bytes([b[p] ^ (1 << rng.randrange(8))]) + b[p + 1:]
    if op == 1:
        return b[:p] + bytes([rng.choice(b'{}[]:,"\\ 0-.eE\x00\x01\xff')]) + b[p + 1:]
    if op == 2:
        return b[:p]
    if op == 3:
        return b[:p] + b[p + 1:]
    return b[:p] + bytes([rng.randrange(256)]) + b[p:]


def test_random_json_and_mutations(parser, oracle):
    rng = random.Random(23)
    for it in range(3000):
        doc = _rand_json(rng).encode()
        if rng.random() < 0.3:
            doc = (" " * rng.randrange(3)).encode() + doc.replace(b",", b" , ")
        check_same(parser, oracle, doc, f"json {it}")
        check_same(parser, oracle, _mutate(rng, doc), f"mut {it}")


def test_configs_small(parser, oracle):
    from tools.gen import generate
    for cfg, size in [(0, 1 << 20), (1, 4 << 20), (2, 4 << 20), (4, 4 << 20)]:
        check_same(parser, oracle, generate(cfg, size), f"C{cfg}")
    nd = generate(3, 1 << 20)
    for k, rec in enumerate(nd.split(b"\n")[:2000]):
        check_same(parser, oracle, rec, f"C3 record {k}")


def test_escape_block_and_tile_boundaries(parser, oracle):
    """Escapes whose sequence or decoded bytes straddle a 64-byte block or a
    16 KiB K1 tile boundary (stage1.cu: spill bytes, overhang_in_scan)."""
    escs = [b"\\n", b"\\u00e9", b"\\u20ac", b"\\ud83d\\ude00", b"\\\\", b"\\u0041"]
    for boundary in (64, 128, 16384, 32768):
        for esc in escs:
            for shift in range(0, 14):
                pos = boundary - shift  # the escape begins here
                head = b'["' + b"b" * (pos - 2)
                doc = head + esc + b"xyz" * 5 + b'", 1]'
                assert doc.index(esc) == pos
                check_same(parser, oracle, doc, f"esc {esc!r} at {boundary}-{shift}")
                # the same escape repeated back to back across the boundary
                doc2 = head + esc * 8 + b'"]'
                check_same(parser, oracle, doc2, f"esc run {esc!r} at {boundary}-{shift}")


def test_escape_decode_in_place_neighbours(parser, oracle):
    """K1 decodes escapes in place in its shared copy of the tile; a block's
    escape window reaching into the next block must see the original bytes.
    An invalid half pair '\\uD83D\\uDC0' ending a block, followed by
    '\\u0030' at the next block's start: decoded in place, the '0' would
    complete the low surrogate (DC00) and hide the STRING_ERROR.  An earlier
    escape in the same block makes the reader's decode come after the
    neighbour's rewrite (a later loop iteration)."""
    for blk in (64, 128, 16384 - 64, 32768 - 64):
        for lead in (b"", b"\\u0041", b"\\u0041\\n\\u00e9"):
            for tail in (b"\\u0030", b"\\u0063", b"\\u0046\\u0030"):
                b = blk + 53  # the half pair occupies the block's last 11 bytes
                mid = b"\\uD83D\\uDC0"
                head = b'["' + b"a" * (b - 2 - len(lead) - 3) + lead + b"bbb"
                doc = head + mid + tail + b'c", 1]'
                assert doc.index(mid) == b and doc.index(tail, b) == blk + 64
                check_same(parser, oracle, doc, f"half pair at {b}, lead {lead!r}, tail {tail!r}")


def _deep_doc(rng, n_items, max_excursion):
    """Containers of both kinds nested past k_stack's 64-kind register, then
    commas, keys and closers back at the outer levels (their container kinds
    were evicted: k_struct looks them up)."""
    out = []

    def value(depth):
        r = rng.random()
        if depth < max_excursion and r < 0.08:  # a deep chain of mixed kinds
            kinds = [rng.choice("{[") for _ in range(rng.randrange(60, max_excursion - depth + 1))]
            for k in kinds:
                out.append('{"k":' if k == "{" else "[")
            out.append(str(rng.randrange(100)))
            for k in reversed(kinds):
                out.append("}" if k == "{" else "]")
        elif r < (0.5 if depth < 3 else 0.25):  # subcritical branching below depth 3
            if rng.random() < 0.5:
                out.append("[")
                for q in range(rng.randrange(1, 5)):
                    if q:
                        out.append(",")
                    value(depth + 1)
                out.append("]")
            else:
                out.append("{")
                for q in range(rng.randrange(1, 5)):
                    if q:
                        out.append(",")
                    out.append('"k%d":' % q)
                    value(depth + 1)
                out.append("}")
        else:
            out.append(rng.choice(['1', '"s"', 'true', 'null', '-2.5e3']))

    out.append("{")
    for q in range(n_items):
        if q:
            out.append(",")
        out.append('"i%d":' % q)
        value(1)
    out.append("}")
    return "".join(out).encode()


def test_deep_nesting_scope(parser, oracle):
    """Token-parallel k_struct at any depth: kinds evicted from k_stack's
    64-kind register (scopeunk) come from the depth tree; closers check their
    kind against the opener found.  Valid documents, kind swaps and stray
    commas / keys after deep excursions, across 4096-token tiles."""
    rng = random.Random(1024)
    for trial in range(40):
        d = _deep_doc(rng, rng.randrange(20, 400), rng.choice([70, 130, 300, 1000]))
        check_same(parser, oracle, d, f"deep {trial}")
        b = bytearray(d)
        for _ in range(3):  # swap a closer's kind / turn a comma into a colon
            k = rng.randrange(len(b))
            while b[k] not in b"}],":
                k = (k + 1) % len(b)
            b[k] = {ord("}"): ord("]"), ord("]"): ord("}"), ord(","): ord(":")}[b[k]]
            check_same(parser, oracle, bytes(b), f"deep {trial} mutated")
    # the same through 2 and 3 emulated shards
    from paper_1902_08318_b200.shard import LocalShards
    for trial in range(6):
        d = _deep_doc(rng, 300, 1000)
        d = d + b" " * ((3 << 14) - len(d)) if len(d) < (3 << 14) else d
        r = oracle.parse(d)
        for G in (2, 3):
            sh = LocalShards(d, G)
            assert sh.run() == (r.name, r.offset), (trial, G)
            if r.code == 0:
                tape, strings = sh.assemble()
                assert np.array_equal(tape, r.tape_array()) and strings == r.strings
            sh.close()


def test_error_sweep(parser, oracle):
    from tools.gen import generate
    for seed in range(1, 200):
        err = 1 + seed % 5
        data = generate(4, 1 << 14, seed=seed, err=err)
        check_same(parser, oracle, data, f"C4 err {err} seed {seed}")


def test_streamed_jt_parse(parser, oracle):
    """jt_parse of documents >= 8 MiB streams the host input in 4 MiB pieces
    (engine.cu parse_stream): stage 1 per piece as it lands, the string
    buffer fetched during stage 2.  Same results as the single-upload path."""
    from tools.gen import generate
    docs = [(generate(1, 20 << 20, seed=3), "C1 20 MiB"), (generate(2, 12 << 20, seed=4), "C2 12 MiB"),
            (generate(4, 18 << 20, seed=5), "C4 18 MiB")]
    base = generate(0, 9 << 20, seed=6)
    # errors late in the document, in the last piece, and a string across a piece boundary
    docs.append((base[:-3] + b"x]", "tail error"))
    k = 4 << 20
    docs.append((base[:k + 5] + b"\xff" + base[k + 6:], "utf-8 error in piece 1"))
    s = b'["' + b"a" * ((8 << 20) + 100) + b'"]'
    docs.append((s, "string across pieces"))
    for data, where in docs:
        check_same(parser, oracle, data, where)


def test_streamed_stage2_ranges(parser, oracle):
    """Streamed jt_parse (stream mode 0) runs stage 2 in token ranges: the
    early ranges while later pieces upload (tape words back early), the last
    one after the upload (engine.cu parse_stream, stage2.cu k_range_a/b).
    Brackets whose opener lies in an earlier range (patches), nesting deeper
    than 64 across ranges, numbers and hard floats in every range, errors in
    early ranges, ranges without tokens, and a tape larger than the early
    host block."""
    from tools.gen import generate
    docs = [(generate(2, 20 << 20, seed=21), "C2 numbers 20 MiB"),
            (generate(0, 24 << 20, seed=22), "C0-style 24 MiB"),
            (b"[" * 1000 + generate(1, 16 << 20, seed=23) + b"]" * 1000, "deep across ranges"),
            (b"{\"a\":" * 60 + generate(4, 16 << 20, seed=24) + b"}" * 60, "objects across ranges")]
    base = generate(1, 16 << 20, seed=25)
    docs.append((base[:3 << 20] + b"}" + base[(3 << 20) + 1:], "error in the first range"))
    docs.append((base[:(9 << 20) + 7] + b"\x01" + base[(9 << 20) + 8:], "control byte mid document"))
    docs.append((b'["' + b"w" * (14 << 20) + b'", [1, 2.5e-310, "x"]]', "early ranges without tokens"))
    docs.append((b"[" + b"1," * (6 << 20) + b"1]", "tape above the early block"))
    docs.append((b"[" + b"1.7976931348623157e308,4.9e-324," * (300000) + b"0]", "hard floats"))
    for data, where in docs:
        check_same(parser, oracle, data, where)
    # jt_parse without a document (out == NULL): code and offset only
    for data, where in docs[:2] + docs[4:6]:
        g, o = parser.parse(data, want_document=False), oracle.parse(data)
        assert (g.name, g.offset) == (o.name, o.offset) and g.document is None, where


def _piece_cut(length: int) -> int:
    """A piece boundary of the streamed jt_parse (engine.cu parse_stream:
    4 MiB pieces, K1 one 16 KiB tile behind each boundary)."""
    return 2 * (4 << 20)


def test_streamed_pieces(parser, oracle):
    """Streamed jt_parse (engine.cu parse_stream): escapes, numbers, atoms
    and brackets across a piece boundary, a piece without a token start, deep
    nesting across pieces, and the resident state (index, jt_stage2) read
    after the streamed parse."""
    from paper_1902_08318_b200 import Parser
    from tools.gen import generate
    parser = Parser()
    n = 12 << 20
    cut = _piece_cut(n)
    filler = generate(0, cut - 4096, seed=11)[1:-1]  # object members of a top-level array
    escs = [b"\\u00e9", b"\\ud83d\\ude00", b"\\n", b"\\\\", b"\\u20ac"]
    for esc in escs:
        for shift in (1, 2, 5, 7, 11):
            head = b"[" + filler + b',"'
            pad = cut - shift - len(head)
            doc = head + b"q" * pad + esc + b'", 1.25e-3, true, {"k": [null]}'
            doc = doc + b"," + generate(0, n - len(doc), seed=12)[1:]
            assert doc.index(esc, len(head)) == cut - shift
            check_same(parser, oracle, doc, f"esc {esc!r} at cut-{shift}")
    for shift in range(1, 24, 3):  # number / atom / bracket tokens straddling the cut
        head = b"[" + filler + b","
        pad = cut - shift - len(head)
        for tok in (b"-12345678901234567.5e-7", b"true", b"null", b"[[]]", b'{"a":{}}'):
            doc = head + b" " * pad + tok + b"," + generate(0, n - cut, seed=13)[1:]
            check_same(parser, oracle, doc, f"token {tok!r} at cut-{shift}")
    # middle pieces without any token start
    s = b'[1,"' + b"z" * (20 << 20) + b'",2]'
    check_same(parser, oracle, s, "token-free piece")
    # nesting deeper than 64 opened in one piece and closed in a later one
    deep = b"[" * 900 + generate(1, 16 << 20, seed=14) + b"]" * 900
    check_same(parser, oracle, deep, "deep across pieces")
    # jt_stage2 after a streamed jt_parse re-uses the retained input + index
    data = generate(1, 10 << 20, seed=15)
    check_same(parser, oracle, data, "C1 10 MiB")
    r = parser.stage2()
    o = oracle.parse(data)
    assert r.name == "OK" and np.array_equal(r.document.tape, o.tape_array())
    assert r.document.strings == o.strings


def test_minify(parser, oracle):
    """jt_minify on the GPU (k_minify) vs the oracle (pinned to the
    reference's jt_minify in test_oracle_vs_ref.py)"""
    from tools.gen import generate
    rng = random.Random(43)
    docs = [b' { "a" : [ 1 , 2 ] } ', b'{"a b": "c \\" d"}', b"[]", b"", b'["a \t b"]', b"[1,]",
            generate(1, 4 << 20), generate(4, 2 << 20), generate(0, 1 << 20), generate(2, 1 << 20),
            generate(1, 9 << 20, seed=8)]
    for _ in range(300):
        d = _rand_json(rng).encode()
        docs += [d, _mutate(rng, d)]
    for d in docs:
        assert parser.minify(d) == oracle.minify(d), d[:120]


def test_stats(parser, oracle):
    """jt_compute_stats on the GPU (k_stats) vs the oracle's restatement
    (pinned to the reference in test_oracle_vs_ref.py)"""
    from tools.gen import generate
    rng = random.Random(53)
    docs = [generate(c, 1 << 20) for c in (0, 1, 2, 4)] + [b"[1,]", b"", b'["\xc3\xa9", -0, 1e5]']
    for _ in range(200):
        d = _rand_json(rng).encode()
        docs += [d, _mutate(rng, d)]
    for d in docs:
        assert parser.stats(d) == oracle.stats(d), d[:120]


def test_document_distinct(parser):
    """jt_document_distinct on GPU-parsed documents vs the reference's own
    (oracle/_ref) on the same input"""
    import os
    from oracle.pyoracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    from tools.gen import generate
    ref = Reference()
    docs = [generate(0, 1 << 18), generate(1, 1 << 18), generate(3, 1 << 16).split(b"\n")[0],
            b'{"a": {"b": [1, 2, 2, -3, 1.5, "x", null, true, {"b": 7}]}, "b": {"a": {"b": false}}}',
            b'[{"k": 1}, {"k": "1"}, {"k": [1.0, 1e300, -0.0, 0]}, {"k": {"k": 9}}]', b"5"]
    rng = random.Random(59)
    for _ in range(150):
        docs.append(_rand_json(rng).encode())
    paths = [b"", b"a", b"b", b"a.b", b"k", b"k.k", b"x.y.z", b"id", b"name", b"b.a.b", b"k0", b"k1.k2", b"k0.k0.k0", b"k3"]
    for d in docs:
        want = ref.distinct(d, paths)
        if want is None:
            continue
        r = parser.parse(d)
        got = [r.document.distinct(p) for p in paths]
        assert got == want, d[:200]
        # the same query selected on the device (jt_b200_distinct)
        assert [parser.distinct(p) for p in paths] == want, d[:200]


def test_device_distinct_large(parser):
    """jt_b200_distinct on full-size synthetic documents (deep trees, many
    matches, long strings) against the host walk of the downloaded document,
    which test_document_distinct pins to the reference"""
    from tools.gen import generate
    for cfg, size in ((0, 1 << 20), (1, 8 << 20), (2, 4 << 20), (4, 8 << 20)):
        d = generate(cfg, size, seed=5 + cfg)
        r = parser.parse(d)
        assert r.name == "OK"
        import re
        keys = [m.group(1) for m in re.finditer(rb'"([^"\\]{1,24})"\s*:', d[:200000])][:40]
        paths = [b"x.y"] + keys[:6] + [a + b"." + b for a, b in zip(keys[:12], keys[1:13])]
        paths += [keys[0] + b"." + keys[1] + b"." + keys[2]] if len(keys) > 2 else []
        hits = 0
        for p in paths:
            want = r.document.distinct(p)
            hits += want.count(b"\n")
            assert parser.distinct(p) == want, (cfg, p)
        assert cfg == 2 or hits > 0, cfg  # C2 has no keys
    assert parser.parse(b"[1, ]").name != "OK"
    assert parser.distinct(b"a") is None  # no successful parse to query


def test_carry_scan_chunk_boundary(parser, oracle):
    """K0b scans the tile functions in chunks of 8192 tiles (128 MiB) with the
    state carried from chunk to chunk: the odd-backslash and in-string carries
    cross that boundary in the middle of a string, both ways (the string ends
    right after it / goes on), and at the last tile before it."""
    B = 8192 * 16384
    for nbs, cut in ((6, B), (7, B), (5, B - 16384), (8, B + 16384)):
        head = b'["' + b"a" * (cut - 2 - nbs // 2)
        doc = head + b"\\" * nbs + b'"' + b"b" * 20000 + (b'"]' if nbs % 2 else b',"c"]')
        assert doc[cut - 1:cut + 1] == b"\\\\"  # the run straddles the boundary
        check_same(parser, oracle, doc, "carry chunk %d %d" % (nbs, cut))
