"""Byte-range sharded parses (shard.h) against the oracle.

G shards are emulated on one GPU (paper_1902_08318_b200.shard.LocalShards):
the same kernels and phase summaries as one-process-per-GPU runs, with the
all-gather replaced by writes into one buffer.  The document result must be
jt_parse's: same error code and offset; on success the concatenated shard
tapes and string buffers equal the oracle's.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TILE = 16384


def check_sharded(oracle, data: bytes, G: int, where=""):
    from paper_1902_08318_b200.shard import LocalShards
    o = oracle.parse(data)
    ls = LocalShards(data, G)
    try:
        name, off = ls.run()
        assert (name, off) == (o.name, o.offset), (where, G, name, off, o.name, o.offset)
        if o.code == 0:
            tape, strings = ls.assemble()
            assert np.array_equal(tape, o.tape_array()), (where, G)
            assert strings == o.strings, (where, G)
    finally:
        ls.close()


def test_shard_layout():
    from paper_1902_08318_b200.shard import layout
    for n, G in [(TILE, 1), (5 * TILE + 7, 3), (64 * TILE, 8), (100 * TILE - 1, 7)]:
        lo = layout(n, G)
        assert lo[0][0] == 0 and lo[-1][1] == n
        assert all(b % TILE == 0 and b < e for b, e in lo)
        assert all(lo[k][1] == lo[k + 1][0] for k in range(G - 1))


def test_shards_configs(oracle):
    from tools.gen import generate
    for cfg, size, Gs in [(0, 1 << 20, (2, 3, 7)), (1, 2 << 20, (2, 5)), (2, 1 << 20, (3,)),
                          (4, 2 << 20, (2, 4, 8))]:
        data = generate(cfg, size)
        for G in Gs:
            check_sharded(oracle, data, G, f"C{cfg}")


def test_shards_error_sweep(oracle):
    from tools.gen import generate
    for seed in range(1, 40):
        err = 1 + seed % 5
        data = generate(4, 1 << 17, seed=seed, err=err)
        G = 2 + seed % 5
        G = min(G, (len(data) + TILE - 1) // TILE)
        check_sharded(oracle, data, G, f"C4 err {err} seed {seed}")


def _pad_array(items: list[bytes], total: int) -> bytes:
    body = b",".join(items)
    return body


def test_shards_crafted(oracle):
    cases = []
    # a string longer than a shard, with escapes and UTF-8 across the cuts
    s = ("ab\\n\\u00e9€\\\"x" * 9000)
    cases.append(('["' + s + '", 1, {"k": "' + s + '"}]').encode())
    # containers opened in shard 0, closed in shard 2; deep (> 64) nesting
    for depth in (3, 70, 900):
        inner = '{"a": [' + ",".join(str(i) for i in range(30000)) + "]}"
        cases.append(("[" * depth + inner + "]" * depth).encode())
        cases.append(('{"x":' * depth + '"' + "y" * 40000 + '"' + "}" * depth).encode())
    # kind mismatch across shards: "[" ... "}"
    cases.append(("[" + "1," * 30000 + "2}").encode())
    # unclosed / overclosed across shards
    cases.append(("[" + "1," * 30000 + "2").encode())
    cases.append(("[" + "1," * 30000 + "2]]").encode())
    # a shard with no token (inside a long string) followed by errors
    cases.append(('["' + "z" * 50000 + '", tru]').encode())
    cases.append(('["' + "z" * 50000 + '\x01"]').encode())
    # UTF-8 error in the last shard beats a grammar error in the first
    cases.append(("[1 2," + "3," * 30000 + '"\xff"]').encode("latin-1"))
    # trailing content / second root across shards
    cases.append(("[" + "1," * 30000 + "2] 3").encode())
    # object keys at the cut
    cases.append(("{" + ",".join(f'"k{i}": {i}' for i in range(12000)) + "}").encode())
    for k, data in enumerate(cases):
        tiles = (len(data) + TILE - 1) // TILE
        for G in sorted({2, 3, min(6, tiles)}):
            if G <= tiles:
                check_sharded(oracle, data, G, f"crafted {k}")


def test_shards_cut_positions(oracle):
    # the same document with its interesting bytes moved across a shard cut
    for shift in range(0, 40, 3):
        head = b'{"a": [' + b"7," * ((TILE - 12 - shift) // 2)
        doc = head + b'"x\\ud83d\\ude00y", {"b": [true, false, null, -1.5e3]}, "\\\\"]}'
        check_sharded(oracle, doc + b" " * 10, 2, f"cut shift {shift}")


def test_shards_deep_then_shallow(oracle):
    """A shard that starts hundreds of levels deep, closes them, then holds
    shallow objects: its own openers are shallow but the carried-in stack is
    not (max depth must include the shard's starting depth)."""
    import os
    deep = '{"a":' * 150 + "[" * 150
    body = "1" + "]" * 150 + "}" * 149
    tail = ', "k": {"x": 1, "y": [1, 2, {"z": "w"}], "v": {"p": true}}' * 600 + "}"
    doc = (deep + "0," * ((TILE - len(deep)) // 2 + 40) + body + tail).encode()
    for G in (2, 3):
        check_sharded(oracle, doc, G, "deep then shallow")
    here = os.path.join(os.path.dirname(__file__), "golden", "fuzz")
    for name in sorted(os.listdir(here)):  # fuzz finds (tests/fuzz_gpu.py)
        data = open(os.path.join(here, name), "rb").read()
        for G in (2, 3, 5):
            if G <= (len(data) + TILE - 1) // TILE:
                check_sharded(oracle, data, G, name)


def test_shards_trailing_token_free(oracle):
    """Shards after the document's last token (a trailing shard inside the
    last number or string): the end-of-input check belongs to the shard that
    holds the last token (fuzz find, tests/fuzz_gpu.py seed 99)."""
    T = 16384
    docs = []
    for tail in (5, 100, T - 1):
        head = b"[" + b"12," * ((2 * T - 8) // 3)
        body = head + b"7" * (2 * T + tail - len(head))  # last number runs into the last shard
        docs.append((body, f"unterminated, number into the last shard (+{tail})"))
        docs.append((body + b"]", f"terminated (+{tail})"))
    docs.append((b"[0." + b"1" * (3 * T), "one number across all shards, unterminated"))
    docs.append((b"0." + b"1" * (3 * T), "root number across all shards"))
    docs.append((b'["' + b"s" * (3 * T), "unterminated string across shards"))
    for data, where in docs:
        for G in (2, 3):
            check_sharded(oracle, data, G, where)
