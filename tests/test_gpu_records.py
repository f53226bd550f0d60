"""NDJSON record mode (BASELINE config C3): every '\\n'-separated record of
one buffer parsed in one GPU pass must give exactly what jt_parse gives for
that record alone (oracle): code, record-relative offset, tape, strings."""
import random

import numpy as np
import pytest

from tests.vectors import KAT

pytestmark = pytest.mark.gpu


def check_records(parser, oracle, data: bytes, where=""):
    import torch
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8) if data else torch.zeros(1, dtype=torch.uint8)
    parser.copy_in(host.data_ptr(), len(data))
    got = parser.parse_records(len(data))
    recs = data.split(b"\n")
    if data.endswith(b"\n"):
        recs = recs[:-1]
    if not data:
        recs = []
    assert len(got) == len(recs), (where, len(got), len(recs))
    for k, (rec, g) in enumerate(zip(recs, got)):
        o = oracle.parse(rec)
        assert (g[0], g[1]) == (o.name, o.offset), (where, k, rec[:120], g[:2], o.name, o.offset)
        if o.code == 0:
            assert np.array_equal(g[2], o.tape_array()), (where, k, rec[:120])
            assert g[3] == o.strings, (where, k)


def test_records_generated(parser, oracle):
    from tools.gen import generate
    for seed in (19023, 5):
        check_records(parser, oracle, generate(3, 1 << 20, seed=seed), f"C3 seed {seed}")


def test_records_kat_lines(parser, oracle):
    # every known-answer vector as one record, in one buffer (no raw '\n' inside)
    lines = [d for d, _, _ in KAT if b"\n" not in d]
    rng = random.Random(7)
    for trial in range(4):
        rng.shuffle(lines)
        buf = b"\n".join(lines) + (b"\n" if trial % 2 else b"")
        check_records(parser, oracle, buf, f"kat trial {trial}")


def test_records_edges(parser, oracle):
    cases = [
        b"", b"\n", b"\n\n", b"1", b"1\n", b"[1,2]\n{}\n", b'"abc\n"def"\n', b'{"a":"x\\\n1}\n',
        b"[[[[\n]]]]\n[1]", b"]\n[\n1\n", b'"\xff"\n"ok"\n', b'"\xe2\x82\n"\n', b"tru\nfalse\nnul",
        b"[1,\n2]", b' {"a": [1, 2, {"b": null}]} \n  \n\t[]\n', b'"a\\u00e9\\ud83d\\ude00"\n"\\u12"\n',
        b"1 2\n3\n", b"{\"k\":1,}\n[1,]\n",
    ]
    for k, c in enumerate(cases):
        check_records(parser, oracle, c, f"edge {k}")


def test_records_long_and_unbalanced(parser, oracle):
    # unbalanced records must not shift later records (segmented depth);
    # records spanning many K1 tiles; strings with escapes across tiles
    rng = random.Random(11)
    lines = []
    for k in range(400):
        m = k % 5
        if m == 0:
            lines.append(b"[" * rng.randrange(1, 60))          # unclosed
        elif m == 1:
            lines.append(b"]" * rng.randrange(1, 5) + b"[1]")   # over-closed
        elif m == 2:
            lines.append(b'{"s": "' + b"\\\\\\\"x" * rng.randrange(1, 3000) + b'", "n": [1.5e3, -2]}')
        elif m == 3:
            lines.append(b"[" + b",".join(b"%d" % rng.randrange(10**9) for _ in range(rng.randrange(1, 4000))) + b"]")
        else:
            lines.append(b'"' + "é€😀".encode() * rng.randrange(1, 2000) + b'"')
    check_records(parser, oracle, b"\n".join(lines) + b"\n", "long/unbalanced")
