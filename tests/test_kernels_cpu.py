"""CPU checks of the sm_100a kernels' per-thread algebra.

The stage-1 block algebra (stage1_block.cuh), the string emission
(strblock.cuh) and the number parser (numparse.cuh) are __host__ __device__
code; these tests compile the very same headers with g++ (tests/cpu_*.cpp)
and compare them with the oracle.  No GPU needed.
"""
import ctypes as C
import os
import random
import struct
import subprocess

import pytest

from tests.test_gpu_parity import _mutate, _rand_json
from tests.vectors import SOUP_POOL

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "_build")


def _lib(name):
    os.makedirs(BUILD, exist_ok=True)
    src = os.path.join(HERE, name + ".cpp")
    out = os.path.join(BUILD, "lib" + name + ".so")
    deps = [src] + [os.path.join(HERE, "..", "paper_1902_08318_b200", "csrc", f)
                    for f in os.listdir(os.path.join(HERE, "..", "paper_1902_08318_b200", "csrc"))]
    if not os.path.exists(out) or any(os.path.getmtime(d) > os.path.getmtime(out) for d in deps):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", src, "-o", out + ".tmp"])
        os.replace(out + ".tmp", out)
    return C.CDLL(out)


@pytest.fixture(scope="module")
def block_lib():
    L = _lib("cpu_block_check")
    L.jt_cpu_stage1.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(C.c_uint32),
                                C.POINTER(C.c_uint64), C.POINTER(C.c_longlong)]
    return L


@pytest.fixture(scope="module")
def string_lib():
    L = _lib("cpu_string_check")
    L.jt_cpu_strings.argtypes = [C.c_char_p, C.c_uint64, C.c_char_p, C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_longlong),
                                 C.POINTER(C.c_int)]
    return L


@pytest.fixture(scope="module")
def number_lib():
    L = _lib("cpu_number_check")
    L.jt_cpu_number.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
    return L


def _stage1(L, d):
    out = (C.c_uint32 * (len(d) + 8))()
    n, u = C.c_uint64(), C.c_longlong()
    mism = L.jt_cpu_stage1(d, len(d), out, C.byref(n), C.byref(u))
    return mism, bytes(out)[:4 * n.value], u.value


def _inputs(rng, k):
    for it in range(k):
        n = rng.randrange(0, 700)
        m = it % 4
        if m == 0:
            yield bytes(rng.choice(SOUP_POOL) for _ in range(n))
        elif m == 1:
            yield bytes(rng.choice([rng.randrange(256), rng.choice(SOUP_POOL), 0x80 + rng.randrange(64),
                                    rng.choice(b"\xc3\xe0\xed\xf0\xf4\xa9\x9f\xa0")]) for _ in range(n))
        elif m == 2:
            yield "".join(rng.choice(["a", "é", "€", "𝄞", '"', "\\", "{", " "]) for _ in range(n // 2)).encode()
        else:
            d = _rand_json(rng).encode()
            yield _mutate(rng, d) if rng.random() < 0.5 else d


def test_stage1_block_algebra(block_lib, oracle):
    rng = random.Random(5)
    for d in _inputs(rng, 6000):
        mism, idx, u = _stage1(block_lib, d)
        assert mism == 0, d  # composed transfer functions == sequential carry
        assert u == oracle.utf8_error_offset(d), d
        if u < 0:
            assert idx == oracle.stage1(d).index, d


def test_utf8_exhaustive_three_bytes(block_lib, oracle):
    # acceptance.cpp:105-154: every 1..3-byte input (sampled leads for length 3)
    for a in range(256):
        for b in range(256):
            d = bytes([a, b])
            assert _stage1(block_lib, d)[2] == oracle.utf8_error_offset(d)
    rng = random.Random(9)
    for _ in range(20000):
        d = bytes([rng.choice(range(0xC0, 0x100)), rng.randrange(256), rng.randrange(256)])
        assert _stage1(block_lib, d)[2] == oracle.utf8_error_offset(d)


def test_string_emission(string_lib, oracle):
    from tools.gen import generate
    rng = random.Random(3)
    docs = [generate(c, 1 << 15, seed=s) for c in (0, 1, 4) for s in (1, 2)]
    docs += [generate(4, 1 << 12, seed=s, err=1 + s % 5) for s in range(100)]
    docs += list(_inputs(rng, 1500))
    # escapes straddling block / 16 KiB tile boundaries (the harness models
    # K1's tiles: spill bytes written by the next tile's first block)
    for boundary in (64, 16384):
        for esc in (b"\\n", b"\\u00e9", b"\\u20ac", b"\\ud83d\\ude00"):
            for shift in range(0, 14):
                head = b'["' + b"b" * (boundary - shift - 2)
                docs += [head + esc + b'xyz", 1]', head + esc * 8 + b'"]']
    # an invalid half pair ending a block before a valid escape (GPU: the
    # neighbour's in-place decode must not be seen, test_gpu_parity)
    for blk in (64, 16384 - 64):
        for tail in (b"\\u0030", b"\\u0046\\u0030"):
            b = blk + 53
            docs.append(b'["' + b"a" * (b - 2 - 9) + b"\\u0041bbb" + b"\\uD83D\\uDC0" + tail + b'c", 1]')
    for d in docs:
        r = oracle.parse(d)
        if r.code == 1:
            continue
        out = C.create_string_buffer(5 * len(d) + 128)
        ol, n, se, ov = C.c_uint64(), C.c_uint64(), C.c_longlong(), C.c_int()
        idx = (C.c_uint32 * (len(d) + 8))()
        aux = (C.c_uint32 * (len(d) + 8))()
        string_lib.jt_cpu_strings(d, len(d), out, C.byref(ol), idx, aux, C.byref(n), C.byref(se),
                                  C.byref(ov))
        assert ov.value == 0, d[:80]
        if r.code == 0:
            assert out.raw[:ol.value] == r.strings, d[:80]
        if r.name == "STRING_ERROR":
            assert se.value == r.offset, d[:80]


def _u(v):
    return b"\\u%04x" % v if v & 1 else b"\\u%04X" % v


def _escape_soup(rng, faulty):
    """A string of escape sequences at a random alignment: valid \\u escapes of every decoded length,
    surrogate pairs, two-byte escapes, plain and UTF-8 bytes; `faulty` adds lone / mismatched
    surrogate halves, bad hex digits, truncated and unknown escapes."""
    good = [lambda: _u(rng.randrange(0, 0x80)), lambda: _u(rng.randrange(0x80, 0x800)),
            lambda: _u(rng.choice([rng.randrange(0x800, 0xD800), rng.randrange(0xE000, 0x10000)])),
            lambda: _u(rng.randrange(0xD800, 0xDC00)) + _u(rng.randrange(0xDC00, 0xE000)),
            lambda: rng.choice([b'\\"', b"\\\\", b"\\/", b"\\b", b"\\f", b"\\n", b"\\r", b"\\t"]),
            lambda: bytes([rng.randrange(0x20, 0x7F)]).replace(b'"', b"d").replace(b"\\", b"D"),
            lambda: rng.choice(["é", "€", "𝄞"]).encode(), lambda: b"\\\\" * rng.randrange(1, 5)]
    bad = [lambda: _u(rng.randrange(0xD800, 0xDC00)), lambda: _u(rng.randrange(0xDC00, 0xE000)),
           lambda: _u(rng.randrange(0xD800, 0xDC00)) + _u(rng.randrange(0, 0xD800)),
           lambda: _u(rng.randrange(0xD800, 0xDC00)) + b"\\n",
           lambda: _u(rng.randrange(0xD800, 0xDC00)) + b"\\uDC0",
           lambda: b"\\u" + bytes(rng.choice(b"0123456789abcdefABCDEFgG:@`/ ") for _ in range(4)),
           lambda: b"\\u" + b"12"[:rng.randrange(0, 3)], lambda: b"\\" + bytes([rng.choice(b"xqU0a ")]),
           lambda: bytes([rng.randrange(0, 0x20)])]
    body = b""
    for _ in range(rng.randrange(1, 40)):
        body += rng.choice(bad)() if faulty and rng.random() < 0.08 else rng.choice(good)()
    pad = b"p" * rng.randrange(0, 140)
    return b'["' + pad + body + b'", "k"]'


def test_escape_soup(string_lib, oracle):
    # the \\u escapes decided from the bit planes (strblock.cuh classify_u) against the oracle's
    # sequential handle_escape: every alignment to the 64-byte blocks, errors at the first failing escape
    rng = random.Random(11)
    n_err = 0
    for it in range(12000):
        d = _escape_soup(rng, it % 2 == 1)
        r = oracle.parse(d)
        out = C.create_string_buffer(5 * len(d) + 128)
        ol, n, se, ov = C.c_uint64(), C.c_uint64(), C.c_longlong(), C.c_int()
        idx = (C.c_uint32 * (len(d) + 8))()
        aux = (C.c_uint32 * (len(d) + 8))()
        string_lib.jt_cpu_strings(d, len(d), out, C.byref(ol), idx, aux, C.byref(n), C.byref(se), C.byref(ov))
        if r.code == 0:
            assert ov.value == 0, d  # (after an error the two overhang computations may differ)
            assert se.value == -1, d
            assert out.raw[:ol.value] == r.strings, d
        else:
            assert r.name == "STRING_ERROR", (r.name, d)
            assert se.value == r.offset, d
            n_err += 1
    assert n_err > 1000


def _rand_number(rng):
    k = rng.randrange(8)
    if k < 3:
        s = ("-" if rng.random() < .5 else "") + str(rng.randrange(1, 10)) + \
            "".join(str(rng.randrange(10)) for _ in range(rng.randrange(0, 18))) + "." + \
            "".join(str(rng.randrange(10)) for _ in range(rng.randrange(1, 19))) + \
            "e" + str(rng.randrange(-330, 320))
    elif k < 5:
        d = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0]
        if d != d or d in (float("inf"), float("-inf")):
            d = 1.5
        s = "%.17g" % d
        if "." not in s and "e" not in s:
            s += ".0"
    elif k < 6:
        s = "".join(str(rng.randrange(10)) for _ in range(rng.randrange(1, 40))).lstrip("0") or "0"
        s += "." + "".join(str(rng.randrange(10)) for _ in range(rng.randrange(1, 400)))
    elif k < 7:
        s = str(rng.randrange(-2 ** 64, 2 ** 64))
    else:
        s = rng.choice(["0.", "1e+", "-.5", "00", "1.5E+10", "1E-5", "-0e0", "1e1e", "0.0e-0",
                        "5e-324", "2.4703282292062328e-324", "1.7976931348623159e308", "1e-400"])
    return s.encode()


def test_numbers_vs_strtod(number_lib, oracle):
    # test_numbers.cpp:134-160 style (exact equality; the reference's own
    # test only demands agreement with MPFR)
    rng = random.Random(23)
    for _ in range(60000):
        t = _rand_number(rng)
        ok, is_int, bits = oracle.number(t)
        b, slow = C.c_uint64(), C.c_int()
        k = number_lib.jt_cpu_number(t + b"\0" * 64, len(t), C.byref(b), C.byref(slow))
        assert (k != 0) == ok, t
        if ok:
            assert (k == 1) == is_int and b.value == bits, t


def test_numbers_digit_runs(number_lib, oracle):
    """8-digit SWAR steps (numparse.cuh): runs around the 8/16/19-digit
    boundaries, leading fraction zeros across chunks, int64 limits"""
    rng = random.Random(29)
    cases = [b"9223372036854775807", b"9223372036854775808", b"-9223372036854775808",
             b"-9223372036854775809", b"12345678", b"123456789012345678", b"1234567890123456789",
             b"12345678901234567890", b"0.00000000000000000001", b"0.000000001234567890123",
             b"0.00000000", b"0.0000000012345678e-5", b"1.0000000000000000000000001"]
    for _ in range(20000):
        ni = rng.choice([0, 1, 7, 8, 9, 11, 12, 16, 17, 19, 20, 25])
        nf = rng.choice([0, 1, 7, 8, 9, 15, 16, 17, 24, 30])
        lz = rng.choice([0, 0, 3, 8, 9, 16, 20])
        ip = (str(rng.randrange(1, 10)) + "".join(rng.choice("0123456789") for _ in range(ni - 1))) if ni else "0"
        fp = "0" * lz + "".join(rng.choice("0123456789") for _ in range(nf))
        t = ip + ("." + fp if fp else "")
        if rng.random() < 0.3:
            t += "e" + rng.choice(["", "-", "+"]) + str(rng.randrange(0, 330))
        if rng.random() < 0.3:
            t = "-" + t
        cases.append(t.encode())
    for t in cases:
        ok, is_int, bits = oracle.number(t)
        b, slow = C.c_uint64(), C.c_int()
        k = number_lib.jt_cpu_number(t + b"\0" * 64, len(t), C.byref(b), C.byref(slow))
        assert (k != 0) == ok, t
        if ok:
            assert (k == 1) == is_int and b.value == bits, t


def test_glibc_subnormal_quirk(number_lib, oracle):
    # (2724151024255084 + 3/4) * 2^-1074: correctly rounded is ...085, glibc
    # strtod (the reference's slow_float) returns ...084; we match glibc.
    from fractions import Fraction
    x = (2724151024255084 + Fraction(3, 4)) * Fraction(2) ** -1074
    num, den = x.numerator, x.denominator
    ip, rem, frac = num // den, num % den, ""
    while rem:
        rem *= 10
        frac += str(rem // den)
        rem %= den
    t = (str(ip) + "." + frac).encode()
    ok, _, bits = oracle.number(t)
    b, slow = C.c_uint64(), C.c_int()
    number_lib.jt_cpu_number(t + b"\0" * 64, len(t), C.byref(b), C.byref(slow))
    assert ok and bits == 2724151024255084 and b.value == bits


def test_atom_register_check(string_lib):
    """k_scalars' atom_ok8 (8 bytes in registers) = atom_ok byte by byte"""
    L = string_lib
    L.jt_cpu_atoms.argtypes = [C.c_char_p, C.c_uint64]
    rng = random.Random(17)
    lits = [b"true", b"false", b"null", b"tru", b"nul", b"fals", b"truex", b"nulll", b"t", b"f", b"n"]
    ends = [b"", b",", b"]", b"}", b" ", b"\n", b"\t", b"\r", b":", b"[", b"{", b'"', b"x", b"0", b"\x00"]
    for _ in range(3000):
        d = b"".join(rng.choice(lits) + rng.choice(ends) for _ in range(rng.randrange(1, 8)))
        assert L.jt_cpu_atoms(d, len(d)) == 0, d
        assert L.jt_cpu_atoms(d, max(0, len(d) - rng.randrange(0, 3))) == 0, d


def test_hex4_swar_exhaustive(string_lib):
    """K1's word-at-a-time \\uXXXX digit decode equals the byte-at-a-time one
    on all 2^32 four-byte words (split in chunks)"""
    L = string_lib
    L.jt_cpu_hex4_check.restype = C.c_uint64
    L.jt_cpu_hex4_check.argtypes = [C.c_uint64, C.c_uint64]
    step = 1 << 30
    for lo in range(0, 1 << 32, step):
        assert L.jt_cpu_hex4_check(lo, lo + step) == 0, hex(lo)
