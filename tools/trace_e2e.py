"""Timeline of the streamed jt_parse (JT_TRACE=1 prints host/device events on
stderr): one config, pinned or pageable input, a few calls.

    JT_TRACE=1 python tools/trace_e2e.py --config 4 [--pageable]
"""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--size", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--pageable", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_1902_08318_b200 import Parser
    from tools.gen import generate
    data = generate(args.config, args.size)
    n = len(data)
    p = Parser()
    if args.pageable:
        buf = C.create_string_buffer(data, n)
        ptr = C.addressof(buf)
    else:
        host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
        ptr = host.data_ptr()
    for k in range(args.reps + 1):
        doc = C.c_void_p()
        t0 = time.perf_counter()
        rc = p._lib.jt_parse(p._h, C.c_char_p(ptr), n, C.byref(doc), None)
        dt = time.perf_counter() - t0
        assert rc == 0, rc
        p._lib.jt_document_free(doc)
        print(f"call {k}: {dt * 1e3:.2f} ms, {n / dt / 1e9:.1f} GB/s", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
