"""Capacity parity (VERDICT r1 "what's missing" 6).

The reference accepts any input below 2^32 bytes (indexer.cpp:33-34) and
sizes its tape and string buffer from the index (tape_builder.cpp:148,152).
The B200 arena is sized from the input length before S is known, so its
bytes per input byte decide the largest document a GPU can take:

  * the footprint after a parse stays within the documented budget
    (engine.cu ensure_stage1 / ensure_stage2: ~35 B per input byte);
  * a 3.5 GiB document parses through jt_parse and equals the UNMODIFIED
    reference's result (oracle/_ref, run on the box) bit for bit;
  * a document whose string buffer reaches 2^32 bytes (u32 offsets between
    the kernels) fails loudly with CAPACITY, offset -1 — the one documented
    deviation: the reference would parse it;
  * len >= 2^32 is CAPACITY, -1 as in the reference.
"""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BUDGET = 36.0  # device bytes per input byte


def test_footprint_per_input_byte():
    from paper_1902_08318_b200 import Parser
    from tools.gen import generate
    d = generate(1, 256 << 20, seed=3)
    p = Parser()
    r = p.parse(d, want_document=False)
    assert r.name == "OK"
    per = p.device_bytes() / len(d)
    assert per <= BUDGET, per
    p.close()


def test_parse_3_5_gib_vs_reference():
    from oracle.pyoracle import Reference
    from paper_1902_08318_b200 import Parser
    from tools.gen import generate
    d = generate(1, 7 << 29, seed=35)  # 3.5 GiB, C1 shape
    assert len(d) >= 7 << 29
    p = Parser()
    r = p.parse(d)
    ref = Reference().parse(d)
    assert (r.name, r.offset) == (ref.name, ref.offset) == ("OK", -1)
    assert p.device_bytes() / len(d) <= BUDGET
    assert hashlib.sha256(r.document.tape.tobytes()).digest() == hashlib.sha256(ref.tape).digest()
    assert hashlib.sha256(r.document.strings).digest() == hashlib.sha256(ref.strings).digest()
    assert np.array_equal(p.index(), np.frombuffer(ref.index, dtype=np.uint32))
    p.close()


def test_string_buffer_past_u32_is_capacity():
    from paper_1902_08318_b200 import Parser
    n = 1_100_000_000  # '"",' x n: string buffer 4 n bytes > 2^32, input 3.3 GB
    d = b"[" + b'"",' * (n - 1) + b'""]'
    p = Parser()
    r = p.parse(d, want_document=False)
    assert (r.name, r.offset) == ("CAPACITY", -1)
    p.close()
