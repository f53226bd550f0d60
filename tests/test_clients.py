"""Compiled C and C++ clients of the drop-in boundary.

tests/clients/test_capi.c restates the reference's proj/tests/test_capi.cpp in
plain C against include/jsontape.h; tests/clients/test_cpp_api.cpp drives the
reference's C++ entry points (jt::build_structural_index / build_tape / parse,
include/jsontape.hpp) the way proj/tests/acceptance.cpp:455-473 does.  Both are
compiled with the system gcc/g++ and linked against libjsontape_b200.so: the
build and link are checked here (no GPU), the binaries run on the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1902_08318_b200")
OUT = os.path.join(ROOT, "tests", "_build")


def _build(src: str, exe: str, cxx: bool) -> str:
    from paper_1902_08318_b200.build import build
    build()
    os.makedirs(OUT, exist_ok=True)
    out = os.path.join(OUT, exe)
    cmd = (["g++", "-std=c++17"] if cxx else ["gcc", "-std=c11"]) + [
        "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "clients", src)]
    if cxx:  # the seeded config generator (tools/jtgen.c) for the generated documents
        from tools.gen import build as build_gen
        tools = os.path.dirname(build_gen())
        cmd += ["-L", tools, "-l:libjtgen.so", "-Wl,-rpath," + tools]
    cmd += ["-L", LIBDIR, "-l:libjsontape_b200.so", "-Wl,-rpath," + LIBDIR, "-o", out]
    subprocess.check_call(cmd)
    return out


def test_c_client_builds():
    assert os.path.exists(_build("test_capi.c", "test_capi", cxx=False))


def test_cpp_client_builds():
    assert os.path.exists(_build("test_cpp_api.cpp", "test_cpp_api", cxx=True))


@pytest.mark.gpu
@pytest.mark.parametrize("src,exe,cxx", [("test_capi.c", "test_capi", False),
                                         ("test_cpp_api.cpp", "test_cpp_api", True)])
def test_client_runs(src, exe, cxx):
    out = _build(src, exe, cxx)
    r = subprocess.run([out], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
