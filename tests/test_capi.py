"""The drop-in boundary: libjsontape_b200.so loads and exports every symbol
include/jsontape.h and include/jsontape_b200.h declare (no GPU needed; no
compute calls here)."""
import ctypes as C
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1902_08318_b200", "libjsontape_b200.so")


def _declared():
    names = set()
    for h in ("jsontape.h", "jsontape_b200.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(jt_\w+)\s*\(", text):
            names.add(m.group(1))
    return names


def test_header_matches_reference_signatures():
    # every entry point of the reference header (proj/include/jsontape.h)
    ref_names = {"jt_parser_new", "jt_parser_free", "jt_parser_set_flags", "jt_parse", "jt_stage1",
                 "jt_index_count", "jt_index_positions", "jt_stage2", "jt_document_free",
                 "jt_document_equal", "jt_document_dump", "jt_document_distinct", "jt_string_free",
                 "jt_minify", "jt_compute_stats", "jt_oracle_validate", "jt_generate",
                 "jt_error_name"}
    assert ref_names <= _declared()


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        from paper_1902_08318_b200.build import build
        build()
    lib = C.CDLL(LIB)
    for name in sorted(_declared()):
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert _declared() <= exported


def test_python_mirror_lists_all_exports():
    from paper_1902_08318_b200.jsontape import EXPORTS
    assert set(EXPORTS) == _declared()


def test_error_names_without_device():
    from paper_1902_08318_b200 import error_name
    assert [error_name(i) for i in range(8)] == ["OK", "UTF8_ERROR", "STRING_ERROR", "NUMBER_ERROR",
                                                 "TAPE_ERROR", "DEPTH_ERROR", "CAPACITY", "EMPTY"]


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        return
    from paper_1902_08318_b200 import Parser
    try:
        Parser()
    except RuntimeError as e:
        assert "CUDA" in str(e)
    else:
        raise AssertionError("parser created without a GPU: that would be a CPU fallback")
