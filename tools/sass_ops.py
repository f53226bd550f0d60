#!/usr/bin/env python3
"""Static SASS opcode histogram per kernel (cuobjdump -sass of an object or library).

  python tools/sass_ops.py paper_1902_08318_b200/build/stage1.o k_index k_carry_fnILb0

Counts are static (instructions in the binary, loops counted once); the ALU/FMA
split follows B300_MICROARCH.md "pipe rates": LOP3/SHF/PRMT/IADD3/ISETP/SEL/... issue
to the ALU pipe, IMAD/FFMA to the FMA pipe.
"""
import collections
import re
import subprocess
import sys

ALU = {"LOP3", "SHF", "PRMT", "IADD3", "IADD", "ISETP", "SEL", "LEA", "IABS", "IMNMX", "VIMNMX", "FLO",
       "BREV", "SGXT", "BMSK", "PLOP3", "ICMP", "VIADD", "MOV", "P2R", "R2P", "LOP", "SHL", "SHR", "IADD32I",
       "VIADDMNMX", "UIADD3"}
FMA = {"IMAD", "FFMA", "FMUL", "FADD", "HFMA2", "IDP"}


def main():
    path, pats = sys.argv[1], sys.argv[2:]
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    fn = None
    hist = collections.defaultdict(collections.Counter)
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d\s+)?([A-Z0-9_]+)", line)
        if m and fn:
            hist[fn][m.group(1)] += 1
    for fn, h in hist.items():
        if pats and not any(p in fn for p in pats):
            continue
        tot = sum(h.values())
        alu = sum(v for k, v in h.items() if k in ALU)
        fma = sum(v for k, v in h.items() if k in FMA)
        print(f"{fn}: total {tot}, ALU-pipe {alu}, FMA-pipe {fma}")
        print("   " + ", ".join(f"{k} {v}" for k, v in h.most_common(18)))


if __name__ == "__main__":
    main()
