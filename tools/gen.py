"""ctypes wrapper for tools/jtgen.c (seeded synthetic configs C0..C4)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libjtgen.so")
SEEDS = {0: 19020, 1: 19021, 2: 19022, 3: 19023, 4: 19024}
SIZES = {0: 1 << 20, 1: 64 << 20, 2: 256 << 20, 3: 1 << 30, 4: 1 << 30}
ERR_KINDS = {1: "invalid UTF-8", 2: "overlong UTF-8", 3: "unbalanced bracket",
             4: "raw control char in string", 5: "bad number"}
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "jtgen.c")
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", src, "-o", SO + ".tmp", "-lm"])
        os.replace(SO + ".tmp", SO)
    return SO


def _load():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.jtg_generate.restype = C.c_void_p
        L.jtg_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_size_t)]
        L.jtg_free.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def generate(config: int, size: int | None = None, seed: int | None = None, err: int = 0) -> bytes:
    L = _load()
    n = C.c_size_t()
    p = L.jtg_generate(config, SIZES[config] if size is None else size,
                       SEEDS[config] if seed is None else seed, err, C.byref(n))
    try:
        # ctypes.string_at takes an int size (< 2 GiB)
        return bytes((C.c_char * n.value).from_address(p)) if n.value else b""
    finally:
        L.jtg_free(p)


def error_injected() -> bool:
    return bool(C.c_int.in_dll(_load(), "jtg_error_injected_last").value)
