"""Python host mirror of the jsontape C ABI (proj/include/jsontape.h), over
the in-tree B200 library libjsontape_b200.so (ctypes, no torch types).

Same names and argument meaning as the reference's C entry points:
``Parser.parse`` <-> jt_parse (capi.cpp:73-93), ``Parser.stage1`` <-> jt_stage1
(95-102), ``Parser.index`` <-> jt_index_count/positions (127-131),
``Parser.stage2`` <-> jt_stage2 (104-125); error codes are jt_error
(jsontape.h:15-24).  Loading fails loudly when the library or a CUDA device is
missing — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libjsontape_b200.so")
# A/B builds: JT_B200_LIB points at another build of the same library
LIB_PATH = os.environ.get("JT_B200_LIB", LIB_PATH)

OK, UTF8_ERROR, STRING_ERROR, NUMBER_ERROR, TAPE_ERROR, DEPTH_ERROR, CAPACITY, EMPTY = range(8)
ERROR_NAMES = ["OK", "UTF8_ERROR", "STRING_ERROR", "NUMBER_ERROR", "TAPE_ERROR", "DEPTH_ERROR",
               "CAPACITY", "EMPTY"]

# every symbol include/jsontape.h and include/jsontape_b200.h declare
EXPORTS = [
    "jt_parser_new", "jt_parser_free", "jt_parser_set_flags", "jt_parse", "jt_stage1",
    "jt_index_count", "jt_index_positions", "jt_stage2", "jt_document_free",
    "jt_document_equal", "jt_document_dump", "jt_document_distinct", "jt_string_free",
    "jt_minify", "jt_compute_stats", "jt_oracle_validate", "jt_generate", "jt_error_name",
    "jt_b200_input_buffer", "jt_b200_stage1_resident", "jt_b200_parse_resident",
    "jt_b200_parse_async", "jt_b200_stage1_async", "jt_b200_finish", "jt_b200_device_index", "jt_b200_device_tape",
    "jt_b200_device_strings", "jt_b200_download", "jt_b200_document_tape", "jt_b200_document_strings", "jt_b200_document_from", "jt_b200_set_stream",
    "jt_b200_last_launches", "jt_b200_device", "jt_b200_last_error", "jt_b200_profile",
    "jt_b200_kernel_times", "jt_b200_copy_in", "jt_b200_distinct", "jt_b200_shard_summary_bytes",
    "jt_b200_shard_begin", "jt_b200_shard_resident", "jt_b200_shard_phase", "jt_b200_shard_finish", "jt_b200_shard_extent",
    "jt_b200_shard_download", "jt_b200_copy_in_range", "jt_b200_parse_records",
    "jt_b200_records", "jt_b200_records_size", "jt_b200_records_download", "jt_b200_device_records", "jt_b200_device_bytes",
]
KERNELS = ["init", "stage1", "tokens", "slow", "tree", "struct", "final"]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load and type the C ABI (no device work happens here)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run __graft_entry__.build() (no CPU fallback)")
    L = C.CDLL(path)
    vp, sz, ll = C.c_void_p, C.c_size_t, C.c_longlong
    L.jt_parser_new.restype = vp
    L.jt_parser_free.argtypes = [vp]
    L.jt_parser_set_flags.argtypes = [vp, C.c_int, C.c_int, C.c_int]
    L.jt_parse.argtypes = [vp, C.c_char_p, sz, C.POINTER(vp), C.POINTER(ll)]
    L.jt_stage1.argtypes = [vp, C.c_char_p, sz, C.POINTER(ll)]
    L.jt_index_count.argtypes = [vp]
    L.jt_index_count.restype = sz
    L.jt_index_positions.argtypes = [vp]
    L.jt_index_positions.restype = C.POINTER(C.c_uint32)
    L.jt_stage2.argtypes = [vp, C.POINTER(vp), C.POINTER(ll)]
    L.jt_document_free.argtypes = [vp]
    L.jt_document_equal.argtypes = [vp, vp]
    L.jt_document_dump.argtypes = [vp]
    L.jt_document_dump.restype = vp
    L.jt_string_free.argtypes = [vp]
    L.jt_error_name.argtypes = [C.c_int]
    L.jt_error_name.restype = C.c_char_p
    L.jt_b200_input_buffer.argtypes = [vp, sz]
    L.jt_b200_input_buffer.restype = vp
    L.jt_b200_stage1_resident.argtypes = [vp, sz, C.POINTER(ll)]
    L.jt_b200_parse_resident.argtypes = [vp, sz, C.POINTER(ll)]
    L.jt_b200_parse_async.argtypes = [vp, sz]
    L.jt_b200_stage1_async.argtypes = [vp, sz]
    L.jt_b200_finish.argtypes = [vp, C.POINTER(ll)]
    L.jt_b200_device_index.argtypes = [vp, C.POINTER(sz)]
    L.jt_b200_device_index.restype = vp
    L.jt_b200_device_tape.argtypes = [vp, C.POINTER(sz)]
    L.jt_b200_device_tape.restype = vp
    L.jt_b200_device_strings.argtypes = [vp, C.POINTER(sz)]
    L.jt_b200_device_strings.restype = vp
    L.jt_b200_download.argtypes = [vp, C.POINTER(vp)]
    L.jt_b200_set_stream.argtypes = [vp, vp]
    L.jt_b200_last_launches.argtypes = [vp]
    L.jt_b200_device.argtypes = [vp]
    L.jt_b200_last_error.argtypes = [vp]
    L.jt_b200_last_error.restype = C.c_char_p
    L.jt_b200_distinct.argtypes = [vp, C.c_char_p]
    L.jt_b200_distinct.restype = vp
    L.jt_b200_profile.argtypes = [vp, C.c_int]
    L.jt_b200_kernel_times.argtypes = [vp, C.POINTER(C.c_float), C.c_int]
    L.jt_b200_copy_in.argtypes = [vp, vp, sz]
    L.jt_b200_shard_summary_bytes.argtypes = [C.c_int]
    L.jt_b200_shard_summary_bytes.restype = sz
    L.jt_b200_shard_begin.argtypes = [vp, sz, C.c_uint, C.c_uint, sz, sz]
    L.jt_b200_shard_resident.argtypes = [vp, sz, sz]
    L.jt_b200_device_bytes.argtypes = [vp]
    L.jt_b200_device_bytes.restype = sz
    L.jt_b200_shard_phase.argtypes = [vp, C.c_int, vp, vp]
    L.jt_b200_shard_finish.argtypes = [vp, vp, C.POINTER(ll)]
    L.jt_b200_shard_extent.argtypes = [vp, C.POINTER(C.c_ulonglong)]
    L.jt_b200_shard_download.argtypes = [vp, vp, vp]
    L.jt_b200_copy_in_range.argtypes = [vp, vp, sz, sz]
    L.jt_minify.argtypes = [vp, C.c_char_p, sz, C.c_char_p, C.POINTER(sz), C.POINTER(ll)]
    L.jt_compute_stats.argtypes = [vp, C.c_char_p, sz, vp, C.POINTER(ll)]
    L.jt_b200_parse_records.argtypes = [vp, sz, C.POINTER(sz)]
    L.jt_b200_records.argtypes = [vp]
    L.jt_b200_records.restype = vp
    L.jt_b200_records_size.argtypes = [vp, C.POINTER(C.c_ulonglong)]
    L.jt_b200_records_download.argtypes = [vp, vp, vp]
    _lib = L
    return L


class JtStats(C.Structure):
    """jt_stats (jsontape.h:71-84)"""
    _fields_ = [(n, C.c_uint64) for n in ("integers", "floats", "strings", "non_ascii_bytes", "objects",
                                           "arrays", "nulls", "trues", "falses", "structurals", "bytes")] + \
               [("bytes_per_structural", C.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def _bytes_at(ptr: int, n: int) -> bytes:
    """ctypes.string_at for any size (its size argument is a C int)"""
    return bytes((C.c_char * n).from_address(ptr)) if n else b""


def error_name(code: int) -> str:
    return load_library().jt_error_name(code).decode()


class Document:
    """Host tape document (jt_document): u64 tape words + string buffer."""

    def __init__(self, handle: int):
        self._h = handle
        self._lib = load_library()

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.jt_document_free(self._h)
            self._h = None

    def _raw(self):
        # jt_document (engine.cu): {u64 *tape; size_t words; u8 *strings; size_t bytes; ...}
        return list((C.c_uint64 * 4).from_address(self._h))

    @property
    def tape(self) -> np.ndarray:
        tp, tn = self._raw()[0:2]
        return np.frombuffer(_bytes_at(tp, tn * 8), dtype=np.uint64) if tn else np.zeros(0, np.uint64)

    @property
    def strings(self) -> bytes:
        sp, sn = self._raw()[2:4]
        return _bytes_at(sp, sn)

    def distinct(self, path: bytes) -> bytes:
        """jt_document_distinct: sorted distinct scalars at a dotted key path"""
        L = self._lib
        L.jt_document_distinct.argtypes = [C.c_void_p, C.c_char_p]
        L.jt_document_distinct.restype = C.c_void_p
        sp = L.jt_document_distinct(self._h, path)
        out = C.string_at(sp)
        L.jt_string_free(sp)
        return out

    def dump(self) -> str:
        s = self._lib.jt_document_dump(self._h)
        out = C.string_at(s).decode("utf-8", "replace")
        self._lib.jt_string_free(s)
        return out

    def __eq__(self, other) -> bool:
        return bool(self._lib.jt_document_equal(self._h, other._h))


@dataclass
class Result:
    code: int
    offset: int
    document: Document | None = None

    @property
    def name(self) -> str:
        return ERROR_NAMES[self.code]


class Parser:
    """jt_parser: one CUDA stream + device arena on the current device."""

    def __init__(self):
        self._lib = load_library()
        self._h = self._lib.jt_parser_new()
        if not self._h:
            raise RuntimeError("jt_parser_new failed: no usable CUDA device")

    def close(self):
        if self._h:
            self._lib.jt_parser_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_flags(self, use_clmul=1, fast_extract=1, vector_classify=1):
        self._lib.jt_parser_set_flags(self._h, use_clmul, fast_extract, vector_classify)

    def parse(self, data: bytes, want_document: bool = True) -> Result:
        doc = C.c_void_p()
        off = C.c_longlong(-7)
        code = self._lib.jt_parse(self._h, data, len(data), C.byref(doc) if want_document else None,
                                  C.byref(off))
        return Result(code, off.value, Document(doc.value) if doc.value else None)

    def stage1(self, data: bytes) -> Result:
        off = C.c_longlong(-7)
        code = self._lib.jt_stage1(self._h, data, len(data), C.byref(off))
        return Result(code, off.value)

    def index(self) -> np.ndarray:
        n = self._lib.jt_index_count(self._h)
        if n == 0:
            return np.zeros(0, np.uint32)
        p = self._lib.jt_index_positions(self._h)
        return np.frombuffer(_bytes_at(C.cast(p, C.c_void_p).value, 4 * n), dtype=np.uint32)

    def stage2(self, want_document: bool = True) -> Result:
        doc = C.c_void_p()
        off = C.c_longlong(-7)
        code = self._lib.jt_stage2(self._h, C.byref(doc) if want_document else None, C.byref(off))
        return Result(code, off.value, Document(doc.value) if doc.value else None)

    # ---- B200 extensions (include/jsontape_b200.h) ----
    def input_buffer(self, n: int) -> int:
        p = self._lib.jt_b200_input_buffer(self._h, n)
        if not p:
            raise MemoryError(self.last_error())
        return p

    def copy_in(self, src_ptr: int, n: int):
        """fill the device input from a host or device pointer"""
        if self._lib.jt_b200_copy_in(self._h, src_ptr, n) != 0:
            raise RuntimeError(self.last_error())

    def parse_resident(self, n: int) -> Result:
        off = C.c_longlong(-7)
        code = self._lib.jt_b200_parse_resident(self._h, n, C.byref(off))
        return Result(code, off.value)

    def stage1_resident(self, n: int) -> Result:
        off = C.c_longlong(-7)
        code = self._lib.jt_b200_stage1_resident(self._h, n, C.byref(off))
        return Result(code, off.value)

    def parse_async(self, n: int) -> int:
        return self._lib.jt_b200_parse_async(self._h, n)

    def stage1_async(self, n: int) -> int:
        return self._lib.jt_b200_stage1_async(self._h, n)

    def finish(self) -> Result:
        off = C.c_longlong(-7)
        code = self._lib.jt_b200_finish(self._h, C.byref(off))
        return Result(code, off.value)

    def download(self) -> Document | None:
        doc = C.c_void_p()
        code = self._lib.jt_b200_download(self._h, C.byref(doc))
        return Document(doc.value) if code == OK and doc.value else None

    def device_tape(self):
        n = C.c_size_t()
        p = self._lib.jt_b200_device_tape(self._h, C.byref(n))
        return p, n.value

    def device_strings(self):
        n = C.c_size_t()
        p = self._lib.jt_b200_device_strings(self._h, C.byref(n))
        return p, n.value

    def device_index(self):
        n = C.c_size_t()
        p = self._lib.jt_b200_device_index(self._h, C.byref(n))
        return p, n.value

    def minify(self, data: bytes):
        """jt_minify: (error name, offset, minified bytes or None)"""
        out = C.create_string_buffer(len(data) + 1)
        n, off = C.c_size_t(), C.c_longlong(-7)
        code = self._lib.jt_minify(self._h, data, len(data), out, C.byref(n), C.byref(off))
        return ERROR_NAMES[code], off.value, (out.raw[:n.value] if code == 0 else None)

    def stats(self, data: bytes):
        """jt_compute_stats: (error name, offset, dict or None)"""
        st = JtStats()
        off = C.c_longlong(-7)
        code = self._lib.jt_compute_stats(self._h, data, len(data), C.addressof(st), C.byref(off))
        return ERROR_NAMES[code], off.value, (st.as_dict() if code == 0 else None)

    RECORD = np.dtype([("code", "<i4"), ("reserved", "<i4"), ("offset", "<i8"), ("tape_begin", "<u8"),
                       ("tape_words", "<u8"), ("string_begin", "<u8"), ("string_bytes", "<u8")])

    def parse_records_arrays(self, n: int, download: bool = True):
        """Parse the n resident bytes as NDJSON records (jt_b200_parse_records).
        Returns (records array of RECORD, tape words, string bytes); the last
        two are None without `download`."""
        cnt = C.c_size_t()
        if self._lib.jt_b200_parse_records(self._h, n, C.byref(cnt)) != 0:
            raise RuntimeError(self.last_error())
        k = cnt.value
        rec = self.RECORD
        arr = np.frombuffer(_bytes_at(self._lib.jt_b200_records(self._h), k * rec.itemsize),
                            dtype=rec) if k else np.zeros(0, rec)
        tape = strings = None
        if download:
            sz = (C.c_ulonglong * 2)()
            self._lib.jt_b200_records_size(self._h, sz)
            tape = np.zeros(max(1, sz[0]), np.uint64)
            sbuf = np.zeros(max(1, sz[1]), np.uint8)
            if self._lib.jt_b200_records_download(self._h, tape.ctypes.data, sbuf.ctypes.data) != 0:
                raise RuntimeError(self.last_error())
            tape = tape[:sz[0]]
            strings = sbuf[:sz[1]]
        return arr, tape, strings

    def parse_records(self, n: int, download: bool = True):
        """Parse the n resident bytes as NDJSON records (jt_b200_parse_records).
        Returns [(name, offset, tape words or None, strings or None)] per record."""
        arr, tape, sarr = self.parse_records_arrays(n, download)
        strings = sarr.tobytes() if sarr is not None else None
        out = []
        for r in arr:
            name = ERROR_NAMES[int(r["code"])]
            if download and name == "OK":
                tb, tw = int(r["tape_begin"]), int(r["tape_words"])
                sb0, sn = int(r["string_begin"]), int(r["string_bytes"])
                out.append((name, int(r["offset"]), tape[tb:tb + tw], strings[sb0:sb0 + sn]))
            else:
                out.append((name, int(r["offset"]), None, None))
        return out

    def distinct(self, path: bytes) -> bytes | None:
        """jt_b200_distinct: distinct_values over the last successful parse,
        selected on the device (same text as Document.distinct)"""
        sp = self._lib.jt_b200_distinct(self._h, path)
        if not sp:
            return None
        out = C.string_at(sp)
        self._lib.jt_string_free(sp)
        return out

    def set_stream(self, stream_handle: int | None):
        self._lib.jt_b200_set_stream(self._h, stream_handle)

    def last_launches(self) -> int:
        return self._lib.jt_b200_last_launches(self._h)

    def profile(self, enable: bool = True):
        self._lib.jt_b200_profile(self._h, 1 if enable else 0)

    def kernel_times(self) -> dict:
        """ms per kernel of the last full parse (needs profile(True))."""
        buf = (C.c_float * 8)()
        n = self._lib.jt_b200_kernel_times(self._h, buf, 8)
        return {KERNELS[k]: buf[k] for k in range(n)}

    def device_bytes(self) -> int:
        """device memory held by this parser's arena"""
        return int(self._lib.jt_b200_device_bytes(self._h))

    def last_error(self) -> str:
        return self._lib.jt_b200_last_error(self._h).decode()
