"""Build libjsontape_b200.so in-tree with nvcc for sm_100a.

python -m paper_1902_08318_b200.build   (or __graft_entry__.build())
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libjsontape_b200.so")
SOURCES = ["stage1.cu", "stage2.cu", "engine.cu"]
HEADERS = ["jt_common.cuh", "shard.h", "stage1_block.cuh", "lookback.cuh", "numparse.cuh", "strparse.cuh",
           "strblock.cuh", "stage1.h", "stage2.h", "pow5_table.inc"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines: tuple = (), lib: str = LIB) -> str:
    """Compile and link.  `defines`/`lib` build an instrumented variant
    (e.g. defines=("JT_TIMELINE",)) next to the product library."""
    objdir = os.path.join(HERE, "build" + "".join("_" + d.lower() for d in defines))
    os.makedirs(objdir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + \
        [os.path.join(ROOT, "include", "jsontape.h"), os.path.join(ROOT, "include", "jsontape_b200.h")]
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = [NVCC] + FLAGS + ["-D" + d for d in defines] + ["-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if verbose or r.returncode:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode:
                raise RuntimeError("nvcc failed for " + src)
    if force or _stale(lib, objs):
        tmp = lib + ".tmp"
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
               "-o", tmp] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
        os.replace(tmp, lib)
    # every symbol the library references must resolve (a kernel launcher
    # left in an anonymous namespace links fine but fails at dlopen)
    r = subprocess.run(["nm", "-C", "--undefined-only", lib], capture_output=True, text=True)
    bad = [l for l in r.stdout.splitlines() if " jt::" in l]
    if bad:
        raise RuntimeError("unresolved symbols in " + lib + ":\n" + "\n".join(bad))
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
