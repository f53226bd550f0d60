"""Do two resident parses on two streams overlap usefully?  Two parsers, each
with its own C4 document of --size bytes: back-to-back on one stream vs
concurrently on two streams (the second started half a parse later, so one's
stage 1 runs next to the other's stage 2).  Aggregate GB/s of both.

    python tools/overlap_probe.py --size 268435456
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--size", type=int, default=256 << 20)
    ap.add_argument("--reps", type=int, default=6)
    args = ap.parse_args()
    import torch
    from paper_1902_08318_b200 import Parser
    from tools.gen import generate
    data = generate(args.config, args.size)
    n = len(data)
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    ps, ss = [], []
    for _ in range(2):
        s = torch.cuda.Stream()
        p = Parser()
        p.set_stream(s.cuda_stream)
        p.copy_in(host.data_ptr(), n)
        ps.append(p)
        ss.append(s)
    torch.cuda.synchronize()
    for p in ps:
        assert p.parse_resident(n).name == "OK"

    def run(concurrent):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.reps):
            if concurrent:
                for p in ps:
                    p.parse_async(n)
                for p in ps:
                    assert p.finish().name == "OK"
            else:
                for p in ps:
                    assert p.parse_resident(n).name == "OK"
        torch.cuda.synchronize()
        return 2 * n * args.reps / (time.perf_counter() - t0) / 1e9

    for _ in range(2):
        print("sequential %.1f GB/s   concurrent %.1f GB/s" % (run(False), run(True)))


if __name__ == "__main__":
    main()
