"""ctypes bindings for the CPU checkers — TEST INFRASTRUCTURE ONLY.

Two checkers live under oracle/:
  * ``Oracle``    — oracle/libjt_oracle.so, the plain-C restatement
                    (oracle/jt_oracle.c) of the reference parse path;
  * ``Reference`` — oracle/_ref/libjsontape_ref.so, the UNMODIFIED reference
                    (/root/reference/proj/src/*.cpp) built by
                    oracle/build_ref.sh, driven through its own C ABI
                    (proj/include/jsontape.h:29-64).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libjt_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libjsontape_ref.so")
REF_DRIVER_SO = os.path.join(HERE, "_ref", "libref_driver.so")

ERROR_NAMES = ["OK", "UTF8_ERROR", "STRING_ERROR", "NUMBER_ERROR", "TAPE_ERROR",
               "DEPTH_ERROR", "CAPACITY", "EMPTY"]


def build_oracle(force: bool = False) -> str:
    """Compile the C restatement (gcc only; runs here and on the GPU box)."""
    src = os.path.join(HERE, "jt_oracle.c")
    if force or not os.path.exists(ORACLE_SO) or \
            os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
        tmp = ORACLE_SO + ".tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared",
                               src, "-o", tmp, "-lm"])
        os.replace(tmp, ORACLE_SO)
    return ORACLE_SO


def build_reference() -> str | None:
    """Build oracle/_ref from /root/reference when the sources are present."""
    subprocess.check_call(["sh", os.path.join(HERE, "build_ref.sh")])
    return REF_SO if os.path.exists(REF_SO) else None


@dataclass
class ParseResult:
    code: int
    offset: int
    index: bytes | None = None       # u32 little-endian positions
    tape: bytes | None = None        # u64 words
    strings: bytes | None = None
    extra: dict = field(default_factory=dict)

    @property
    def name(self) -> str:
        return ERROR_NAMES[self.code]

    def index_list(self):
        import numpy as np
        return np.frombuffer(self.index or b"", dtype=np.uint32)

    def tape_array(self):
        import numpy as np
        return np.frombuffer(self.tape or b"", dtype=np.uint64)


class _JtoResult(C.Structure):
    _fields_ = [("code", C.c_int), ("offset", C.c_longlong),
                ("index", C.POINTER(C.c_uint32)), ("index_count", C.c_size_t),
                ("tape", C.POINTER(C.c_uint64)), ("tape_len", C.c_size_t),
                ("strings", C.POINTER(C.c_uint8)), ("strings_len", C.c_size_t)]


class Oracle:
    """The plain-C restatement (oracle/jt_oracle.c)."""

    def __init__(self):
        self.lib = C.CDLL(build_oracle())
        L = self.lib
        L.jto_parse.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(_JtoResult)]
        L.jto_stage1.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(_JtoResult)]
        L.jto_free.argtypes = [C.POINTER(_JtoResult)]
        L.jto_minify.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.POINTER(C.c_size_t),
                                 C.POINTER(C.c_longlong)]
        L.jto_utf8_error_offset.argtypes = [C.c_char_p, C.c_size_t]
        L.jto_utf8_error_offset.restype = C.c_longlong
        L.jto_parse_number.argtypes = [C.c_char_p, C.c_size_t, C.c_size_t,
                                       C.POINTER(C.c_int), C.POINTER(C.c_uint64)]
        L.jto_parse_string.argtypes = [C.c_char_p, C.c_size_t, C.c_size_t,
                                       C.c_char_p, C.POINTER(C.c_uint32),
                                       C.POINTER(C.c_longlong)]

    def minify(self, data: bytes):
        """(error name, offset, minified bytes or None) as jt_minify"""
        out = C.create_string_buffer(len(data) + 1)
        n, off = C.c_size_t(), C.c_longlong()
        code = self.lib.jto_minify(data, len(data), out, C.byref(n), C.byref(off))
        return ERROR_NAMES[code], off.value, (out.raw[:n.value] if code == 0 else None)

    def stats(self, data: bytes):
        """jt_compute_stats restated over the oracle's tape (stats.cpp:5-47)"""
        r = self.parse(data)
        if r.code != 0:
            return ERROR_NAMES[r.code], r.offset, None
        import numpy as np
        t = r.tape_array()
        s = dict(integers=0, floats=0, strings=0, non_ascii_bytes=sum(b >= 0x80 for b in data),
                 objects=0, arrays=0, nulls=0, trues=0, falses=0)
        tags = {ord("l"): "integers", ord("d"): "floats", ord('"'): "strings", ord("{"): "objects",
                ord("["): "arrays", ord("n"): "nulls", ord("t"): "trues", ord("f"): "falses"}
        i = 0
        while i < len(t):
            tag = int(t[i]) >> 56
            if tag in tags:
                s[tags[tag]] += 1
            i += 2 if tag in (ord("l"), ord("d")) else 1
        s["structurals"] = len(r.index_list())
        s["bytes"] = len(data)
        s["bytes_per_structural"] = len(data) / s["structurals"] if s["structurals"] else 0.0
        return "OK", -1, s

    def parse(self, data: bytes) -> ParseResult:
        r = _JtoResult()
        self.lib.jto_parse(data, len(data), C.byref(r))
        out = ParseResult(r.code, r.offset)
        if r.index:
            out.index = C.string_at(r.index, 4 * r.index_count)
        if r.code == 0:
            out.tape = C.string_at(r.tape, 8 * r.tape_len)
            out.strings = C.string_at(r.strings, r.strings_len) if r.strings_len else b""
        self.lib.jto_free(C.byref(r))
        return out

    def stage1(self, data: bytes) -> ParseResult:
        r = _JtoResult()
        self.lib.jto_stage1(data, len(data), C.byref(r))
        out = ParseResult(r.code, r.offset)
        if r.code == 0:
            out.index = C.string_at(r.index, 4 * r.index_count) if r.index_count else b""
        self.lib.jto_free(C.byref(r))
        return out

    def utf8_error_offset(self, data: bytes) -> int:
        return self.lib.jto_utf8_error_offset(data, len(data))

    def number(self, text: bytes):
        """(ok, is_integer, raw 64-bit word) of parse_number on a padded token."""
        buf = text + b"\0" * 64
        is_int = C.c_int(0)
        bits = C.c_uint64(0)
        ok = self.lib.jto_parse_number(buf, len(text), 0, C.byref(is_int), C.byref(bits))
        return bool(ok), bool(is_int.value), bits.value

    def string(self, text: bytes):
        """(ok, decoded bytes or None, error offset) of parse_string at 0."""
        buf = text + b"\0" * 64
        dst = C.create_string_buffer(len(text) + 64)
        n = C.c_uint32(0)
        e = C.c_longlong(-1)
        ok = self.lib.jto_parse_string(buf, len(text), 0, dst, C.byref(n), C.byref(e))
        if ok:
            return True, dst.raw[4:4 + n.value], -1
        return False, None, e.value


class RefDriver:
    """oracle/ref_driver.c: the reference's jt_parse timed on `threads`
    pthreads (one jt_parser each), for bench.py's CPU baseline."""

    def __init__(self, path: str = REF_DRIVER_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.jtref_parse_many.restype = C.c_double
        L.jtref_parse_many.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.jtref_parse_records.restype = C.c_double
        L.jtref_parse_records.argtypes = [C.c_char_p, C.c_size_t, C.c_int, C.c_int,
                                          C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]

    def parse_many(self, data: bytes, threads: int, reps: int) -> tuple[float, int]:
        """(wall seconds of `reps` jt_parse of `data` on each of `threads`
        threads, code of the last parse)"""
        code = C.c_int(-1)
        dt = self.lib.jtref_parse_many(data, len(data), threads, reps, C.byref(code))
        if dt < 0:
            raise RuntimeError("jtref_parse_many failed")
        return dt, code.value

    def parse_records(self, data: bytes, threads: int, reps: int) -> tuple[float, int, int]:
        """(wall seconds of `reps` passes over the '\n'-separated records,
        each jt_parse()d alone, dealt to `threads` threads; records; OK)"""
        nr, ok = C.c_size_t(), C.c_size_t()
        dt = self.lib.jtref_parse_records(data, len(data), threads, reps, C.byref(nr), C.byref(ok))
        if dt < 0:
            raise RuntimeError("jtref_parse_records failed")
        return dt, nr.value, ok.value


class Reference:
    """The unmodified reference through its own C ABI (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        L.jt_parser_new.restype = C.c_void_p
        L.jt_parser_free.argtypes = [C.c_void_p]
        L.jt_parse.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t,
                               C.POINTER(C.c_void_p), C.POINTER(C.c_longlong)]
        L.jt_stage1.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t,
                                C.POINTER(C.c_longlong)]
        L.jt_stage2.argtypes = [C.c_void_p, C.POINTER(C.c_void_p),
                                C.POINTER(C.c_longlong)]
        L.jt_index_count.argtypes = [C.c_void_p]
        L.jt_index_count.restype = C.c_size_t
        L.jt_index_positions.argtypes = [C.c_void_p]
        L.jt_index_positions.restype = C.POINTER(C.c_uint32)
        L.jt_document_free.argtypes = [C.c_void_p]
        L.jt_document_dump.argtypes = [C.c_void_p]
        L.jt_document_dump.restype = C.c_void_p
        L.jt_string_free.argtypes = [C.c_void_p]
        self.p = L.jt_parser_new()

    def __del__(self):
        try:
            self.lib.jt_parser_free(self.p)
        except Exception:
            pass

    def parse_code(self, data: bytes):
        off = C.c_longlong(-7)
        code = self.lib.jt_parse(self.p, data, len(data), None, C.byref(off))
        return code, off.value

    def stats(self, data: bytes):
        """the reference's jt_compute_stats (capi.cpp:169-191)"""
        from paper_1902_08318_b200.jsontape import JtStats
        L = self.lib
        L.jt_compute_stats.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, C.c_void_p,
                                       C.POINTER(C.c_longlong)]
        st = JtStats()
        off = C.c_longlong(-7)
        code = L.jt_compute_stats(self.p, data, len(data), C.addressof(st), C.byref(off))
        return ERROR_NAMES[code], off.value, (st.as_dict() if code == 0 else None)

    def minify(self, data: bytes):
        """the reference's jt_minify (capi.cpp:154-167)"""
        L = self.lib
        L.jt_minify.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t, C.c_char_p,
                                C.POINTER(C.c_size_t), C.POINTER(C.c_longlong)]
        out = C.create_string_buffer(len(data) + 1)
        n, off = C.c_size_t(), C.c_longlong(-7)
        code = L.jt_minify(self.p, data, len(data), out, C.byref(n), C.byref(off))
        return ERROR_NAMES[code], off.value, (out.raw[:n.value] if code == 0 else None)

    def stage1(self, data: bytes) -> ParseResult:
        off = C.c_longlong(-7)
        code = self.lib.jt_stage1(self.p, data, len(data), C.byref(off))
        out = ParseResult(code, off.value)
        if code == 0:
            n = self.lib.jt_index_count(self.p)
            out.index = _bytes_at(C.cast(self.lib.jt_index_positions(self.p), C.c_void_p).value, 4 * n) if n else b""
        return out

    def distinct(self, data: bytes, paths):
        """the reference's jt_document_distinct for each path (None if the parse fails)"""
        L = self.lib
        L.jt_document_distinct.argtypes = [C.c_void_p, C.c_char_p]
        L.jt_document_distinct.restype = C.c_void_p
        doc = C.c_void_p()
        off = C.c_longlong(-7)
        if self.lib.jt_parse(self.p, data, len(data), C.byref(doc), C.byref(off)) != 0:
            return None
        out = []
        for path in paths:
            sp = L.jt_document_distinct(doc, path)
            out.append(C.string_at(sp))
            L.jt_string_free(sp)
        L.jt_document_free(doc)
        return out

    def parse(self, data: bytes) -> ParseResult:
        """Full parse; tape words and strings recovered from the reference's
        own document dump is lossy, so the tape is read through the
        jt_document struct layout instead (see _doc_words)."""
        doc = C.c_void_p()
        off = C.c_longlong(-7)
        code = self.lib.jt_parse(self.p, data, len(data), C.byref(doc), C.byref(off))
        out = ParseResult(code, off.value)
        n = self.lib.jt_index_count(self.p)
        if code != 1:  # index is refreshed unless stage 1 failed on UTF-8
            out.index = _bytes_at(C.cast(self.lib.jt_index_positions(self.p), C.c_void_p).value, 4 * n) if n else b""
        if code == 0:
            out.tape, out.strings = _doc_words(doc.value)
            self.lib.jt_document_free(doc)
        return out


def _bytes_at(ptr: int, n: int) -> bytes:
    """ctypes.string_at for any size (its size argument is a C int)"""
    return bytes((C.c_char * n).from_address(ptr)) if n else b""


def _doc_words(doc_ptr: int):
    """jt_document{parsed_document{raw_vector<u64> tape; raw_vector<u8>
    strings; size_t source_length}} (proj/src/capi.cpp:21-23, tape.h:49-58):
    two libstdc++ std::vector triples (begin, end, cap)."""
    words = (C.c_uint64 * 6).from_address(doc_ptr)
    tb, te, _, sb, se, _ = list(words)
    tape = _bytes_at(tb, te - tb) if te > tb else b""
    strings = _bytes_at(sb, se - sb) if se > sb else b""
    return tape, strings
