"""ncu driver for the end-to-end path: jt_parse (host input, streamed
pieces for documents >= 8 MiB) of one config, `--reps` times after one
warm-up call (python tools/prof_e2e.py --config 1)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--size", type=int, default=None)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    import torch
    from paper_1902_08318_b200 import Parser
    from tools.gen import generate
    data = generate(args.config, args.size)
    p = Parser()
    for _ in range(1 + args.reps):
        r = p.parse(data)
        assert r.name == "OK", r.name
    torch.cuda.synchronize()
    print("ok", len(data))


if __name__ == "__main__":
    main()
