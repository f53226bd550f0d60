"""Minimal driver for ncu captures: one resident full parse and one resident
jt_stage1 of a config, nothing else (python tools/prof.py --config 1)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--size", type=int, default=None)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--mode", default="both", choices=["both", "parse", "stage1"])
    args = ap.parse_args()
    import torch
    from paper_1902_08318_b200 import Parser
    from tools.gen import generate
    data = generate(args.config, args.size)
    n = len(data)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    p = Parser()
    p.set_stream(s.cuda_stream)
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    p.copy_in(host.data_ptr(), n)
    torch.cuda.synchronize()
    for _ in range(args.reps):
        if args.mode in ("both", "parse"):
            r = p.parse_resident(n)
            assert r.name == "OK", r.name
        if args.mode in ("both", "stage1"):
            r = p.stage1_resident(n)
            assert r.name == "OK", r.name
    torch.cuda.synchronize()
    print("ok", n)


if __name__ == "__main__":
    main()
