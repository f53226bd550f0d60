"""K1 per-tile phase timeline (JT_TIMELINE build, %globaltimer stamps by
thread 0 and the warps' arrivals at the barrier after the weight scans).

    python -c "from paper_1902_08318_b200.build import build; build(defines=('JT_TIMELINE',), \
        lib='paper_1902_08318_b200/ab_timeline.so')"
    JT_B200_LIB=$PWD/paper_1902_08318_b200/ab_timeline.so python tools/k1_timeline.py --config 4

Stamps (stage1.cu): 0 start, 1 after the count-scan barrier, 2 after the
weight-scan barrier (10-15: warps 0-5 arriving there), 6 staging starts, 8
warp 0's staging done, 5 its look-back done, 3 after the staging barrier, 9 after the length-field
barrier, 7 end.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--size", type=int, default=None)
    args = ap.parse_args()
    import torch
    from paper_1902_08318_b200 import Parser
    from tools.gen import generate
    data = generate(args.config, args.size)
    n = len(data)
    ntiles = (n + 16383) // 16384
    p = Parser()
    p._lib.jt_b200_timeline.argtypes = [C.c_void_p, C.c_size_t]
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8).pin_memory()
    p.copy_in(host.data_ptr(), n)
    assert p.parse_resident(n).name == "OK"
    buf = np.zeros(min(ntiles, 1 << 17) * 16, dtype=np.uint64)
    p._lib.jt_b200_timeline(buf.ctypes.data, buf.size)  # discard (reset)
    assert p.parse_resident(n).name == "OK"
    p._lib.jt_b200_timeline(buf.ctypes.data, buf.size)
    t = buf.reshape(-1, 16).astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    names = [(0, 1, "load, classify, UTF-8, escape overhang, count scan"),
             (1, 2, "escape weights + in-place decode, weight scans (barrier)"),
             (2, 6, "publish aggregate"),
             (6, 8, "warp 0: its staging copy"),
             (8, 5, "warp 0: look-back (predecessors' counts)"),
             (5, 3, "wait for the other warps' staging (barrier)"),
             (3, 9, "copy-out of index / aux / tok / tape_idx + lengths"),
             (9, 7, "payload copy-out")]
    print(f"config {args.config}: {len(t)} tiles, span {(t[:, 7].max() - t0) / 1e3:.1f} us")
    for a, b, what in names:
        d = (t[:, b] - t[:, a]).astype(np.float64)
        print(f"  {a}->{b} {what:58s} median {np.median(d):8.0f} ns  mean {d.mean():8.0f}  p90 {np.percentile(d, 90):8.0f}")
    life = (t[:, 7] - t[:, 0]).astype(np.float64)
    print(f"  lifetime median {np.median(life):.0f} ns, mean {life.mean():.0f}")
    arr = t[:, 10:16]
    spread = (arr.max(axis=1) - arr.min(axis=1)).astype(np.float64)
    wait = (t[:, 2] - arr.min(axis=1)).astype(np.float64)
    print(f"  weight-scan barrier: arrival spread of warps 0-5 median {np.median(spread):.0f} ns, "
          f"mean {spread.mean():.0f}; first arrival to release median {np.median(wait):.0f} ns")


if __name__ == "__main__":
    main()
