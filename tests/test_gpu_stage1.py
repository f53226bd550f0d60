"""jt_stage1 (k_index: UTF-8 check + structural index, no stage-2 arrays)
against the oracle's stage 1, and jt_stage2 after it against the oracle's
full parse (include/jsontape_b200.h jt_stage1/jt_stage2; reference
proj/include/jsontape.h jt_stage1/jt_stage2, indexer.cpp build_structural_index).
"""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TILE = 16384


def check_stage1(parser, oracle, data: bytes, where=""):
    g = parser.stage1(data)
    o = oracle.stage1(data)
    assert (g.name, g.offset) == (o.name, o.offset), (where, len(data))
    if o.code == 0:
        assert np.array_equal(parser.index(), o.index_list()), (where, len(data))
    return g


def check_then_stage2(parser, oracle, data: bytes, where=""):
    g = check_stage1(parser, oracle, data, where)
    if g.name != "OK":
        return
    o = oracle.parse(data)
    r = parser.stage2()
    assert (r.name, r.offset) == (o.name, o.offset), (where, len(data))
    if o.code == 0:
        assert np.array_equal(r.document.tape, o.tape_array()), where
        assert r.document.strings == o.strings, where
    # a second jt_stage2 over the same index re-runs stage 2 only
    r2 = parser.stage2()
    assert (r2.name, r2.offset) == (o.name, o.offset), where


def test_stage1_configs(parser, oracle):
    from tools.gen import generate
    for cfg in (0, 1, 2, 3, 4):
        for size in (1000, TILE - 1, TILE, TILE + 1, 5 * TILE + 77, 1 << 20, 3 << 20):
            check_stage1(parser, oracle, generate(cfg, size, seed=size + cfg), f"C{cfg} {size}")


def test_stage1_then_stage2_configs(parser, oracle):
    from tools.gen import generate
    for cfg in (0, 1, 2, 4):
        for size in (5000, 3 * TILE + 5, 1 << 20):
            check_then_stage2(parser, oracle, generate(cfg, size, seed=7 + cfg), f"C{cfg} {size}")


def test_stage1_errors(parser, oracle):
    from tools.gen import generate
    for seed in range(1, 30):
        data = generate(4, 1 << 16, seed=seed, err=1 + seed % 5)
        check_then_stage2(parser, oracle, data, f"err seed {seed}")


def test_stage1_utf8_and_strings(parser, oracle):
    rng = random.Random(5)
    pieces = [b'"', b"\\", b'\\"', b"\\u00e9", b"\xc3\xa9", b"\xe2\x82\xac", b"\xf0\x9f\x98\x80",
              b"\xff", b"\xc3", b"\xed\xa0\x80", b"a", b" ", b"[", b"]", b"{", b"}", b":", b","]
    for it in range(400):
        n = rng.choice([10, 200, TILE - 3, TILE + 40, 2 * TILE + 9])
        out = bytearray()
        while len(out) < n:
            out += rng.choice(pieces) if rng.random() < 0.3 else b"x" * rng.randrange(1, 60)
        data = bytes(out)
        check_stage1(parser, oracle, data, f"soup {it}")


def test_stage1_mutations(parser, oracle):
    from tests.test_gpu_parity import _mutate, _rand_json
    rng = random.Random(99)
    for it in range(300):
        d = b"[" + b",".join(_rand_json(rng).encode() for _ in range(rng.randrange(1, 60))) + b"]"
        for _ in range(rng.randrange(0, 3)):
            d = _mutate(rng, d)
        check_then_stage2(parser, oracle, d, f"mut {it}")


def test_stage1_then_parse_interleaved(parser, oracle):
    """jt_parse after an index-only jt_stage1 must not reuse its state"""
    from tools.gen import generate
    a = generate(1, 1 << 18, seed=3)
    b = generate(2, 1 << 18, seed=4)
    check_stage1(parser, oracle, a, "a")
    g = parser.parse(b)
    o = oracle.parse(b)
    assert (g.name, g.offset) == (o.name, o.offset)
    assert np.array_equal(g.document.tape, o.tape_array())
    check_then_stage2(parser, oracle, a, "a again")


def test_stage1_empty_and_whitespace(parser, oracle):
    for data in (b"", b" ", b"\n\t ", b"1", b'"', b"\\", b"\xff"):
        check_stage1(parser, oracle, data, repr(data))


def test_stage1_many_tiles_per_cta(parser, oracle):
    """documents with far more tiles than resident CTAs (the persistent
    k_index loops over tiles, overlapping each tile's look-back with the
    next tile), incl. tiles past the 4096-entry staging capacity"""
    from tools.gen import generate
    for cfg, size in ((1, 40 << 20), (4, 24 << 20), (2, 20 << 20), (0, 9 << 20)):
        check_stage1(parser, oracle, generate(cfg, size, seed=11 + cfg), f"C{cfg} {size}")
    dense = b"[" + b"1," * (4 << 20) + b"1]"
    check_stage1(parser, oracle, dense, "dense")
    mixed = b"[" + b",".join([b"1," * 3000 + b'"' + b"x" * 20000 + b'"'] * 300) + b"]"
    check_stage1(parser, oracle, mixed, "mixed")
