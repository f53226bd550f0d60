"""Bit-exact parity at the BASELINE.json sizes (VERDICT r1 "what's missing" 1).

Every config document is regenerated on the box (tools/jtgen.c, seeds of
tools.gen.SEEDS) and compared, by sha256, with what the UNMODIFIED reference
produced for it here (tests/golden/large_outputs.json, made by
tests/golden/make_golden_large.py from oracle/_ref):

  * C0 1 MiB, C1 64 MiB, C2 256 MiB, C4 1 GiB through the public jt_parse
    (host buffer in, host document out: the streamed path for >= 8 MiB), the
    device-resident parse + download, and jt_stage1 (k_index): code, offset,
    structural index, tape words (float64 bit patterns included), strings;
  * 8 single-error variants of the C4 document with the error past byte 2^30
    (invalid / overlong UTF-8, mismatched and unbalanced brackets, raw control
    bytes in strings, bad numbers): code, offset and the index the reference
    leaves behind;
  * C3 1 GiB NDJSON (3.9M records), each record as jt_parse(record): per-record
    code and offset, and every OK record's tape and strings, in one GPU pass.
"""
import numpy as np
import pytest

from tests.large_cases import CLEAN, document, gather_ranges, load_fixture, mutate, record_digest, sha

pytestmark = pytest.mark.gpu

FIX = load_fixture()
ROWS = {r["name"]: r for r in FIX["clean"]}


def _pinned(data: bytes):
    import torch
    return torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()


@pytest.mark.parametrize("name", [n for n, _, _ in CLEAN])
def test_large_clean(parser, name):
    row = ROWS[name]
    d = document(row["config"])
    assert len(d) == row["bytes"] and sha(d) == row["input_sha"], "generator drifted on this box"
    # the drop-in entry point: pageable host bytes -> host document
    r = parser.parse(d)
    assert (r.name, r.offset) == (row["code"], row["offset"])
    idx = parser.index()
    assert len(idx) == row["S"] and sha(idx.tobytes()) == row["index_sha"]
    tape = r.document.tape
    assert len(tape) == row["T"] and sha(tape.tobytes()) == row["tape_sha"]
    s = r.document.strings
    assert len(s) == row["string_bytes"] and sha(s) == row["strings_sha"]
    del r, tape, s
    # device-resident parse (the bench's `value` path) + download
    host = _pinned(d)
    parser.copy_in(host.data_ptr(), len(d))
    rr = parser.parse_resident(len(d))
    assert (rr.name, rr.offset) == (row["code"], row["offset"])
    doc = parser.download()
    assert sha(doc.tape.tobytes()) == row["tape_sha"] and sha(doc.strings) == row["strings_sha"]
    del doc
    # jt_stage1 alone (k_index): the reference's stage-1 index
    r1 = parser.stage1(d)
    assert r1.name == "OK"
    assert sha(parser.index().tobytes()) == row["index_sha"]


@pytest.mark.parametrize("k", range(len(FIX["errors"])))
def test_large_error_variants(parser, k):
    row = FIX["errors"][k]
    assert row["patch"][0] >= 1 << 30
    d = mutate(document(4), row["patch"])
    r = parser.parse(d, want_document=False)
    assert (r.name, r.offset) == (row["code"], row["offset"]), row["name"]
    if row["code"] != "UTF8_ERROR":
        idx = parser.index()
        assert len(idx) == row["S"] and sha(idx.tobytes()) == row["index_sha"], row["name"]
    # the resident path agrees
    host = _pinned(d)
    parser.copy_in(host.data_ptr(), len(d))
    rr = parser.parse_resident(len(d))
    assert (rr.name, rr.offset) == (row["code"], row["offset"]), row["name"]


def test_large_records():
    from paper_1902_08318_b200 import Parser
    row = FIX["records"]
    d = document(row["config"])
    assert len(d) == row["bytes"] and sha(d) == row["input_sha"]
    p = Parser()
    host = _pinned(d)
    p.copy_in(host.data_ptr(), len(d))
    arr, tape, strings = p.parse_records_arrays(len(d))
    ok = arr["code"] == 0
    tape_ok = gather_ranges(tape, arr["tape_begin"][ok], arr["tape_words"][ok])
    str_ok = gather_ranges(strings, arr["string_begin"][ok], arr["string_bytes"][ok])
    got = record_digest(arr["code"], arr["offset"], tape_ok.tobytes(), str_ok.tobytes())
    for key in ("records", "ok", "codes_sha", "offsets_sha", "tape_sha", "strings_sha"):
        assert got[key] == row[key], key
    p.close()
