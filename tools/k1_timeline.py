"""K1 per-tile phase timeline (JT_TIMELINE build, %globaltimer stamps by
thread 0 and the warps' arrivals at the barrier after the weight scans).

    python -c "from paper_1902_08318_b200.build import build; build(defines=('JT_TIMELINE',), \
        lib='paper_1902_08318_b200/ab_timeline.so')"
    JT_B200_LIB=$PWD/paper_1902_08318_b200/ab_timeline.so python tools/k1_timeline.py --config 4

Stamps (stage1.cu): 0 start, 1 after the count-scan barrier, 2 after the
weight-scan barrier, 6 staging starts, 8 warp 0's staging done (10-15: warps
0-5 done staging), 5 the look-back done (by the first warp done staging), 3
after the staging barrier, 9 after the length-field barrier, 7 end.
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
    names = [(0, 1, "load, classify, UTF-8, escape classes, count scan (barrier)"),
             (1, 2, "weights, weight scans (barrier)"),
             (2, 6, "publish aggregate"),
             (6, 8, "warp 0: in-place decode + staging copy"),
             (3, 9, "copy-out of index / aux / tok / tape_idx + lengths"),
             (9, 7, "payload copy-out")]
    print(f"config {args.config}: {len(t)} tiles, span {(t[:, 7].max() - t0) / 1e3:.1f} us")
    for a, b, what in names:
        d = (t[:, b] - t[:, a]).astype(np.float64)
        print(f"  {a}->{b} {what:58s} median {np.median(d):8.0f} ns  mean {d.mean():8.0f}  p90 {np.percentile(d, 90):8.0f}")
    life = (t[:, 7] - t[:, 0]).astype(np.float64)
    print(f"  lifetime median {np.median(life):.0f} ns, mean {life.mean():.0f}")
    # the barrier after the staging: released when the last warp has staged AND
    # the look-back (run by the first warp done staging) has the tile's base
    arr = t[:, 10:16]                      # warps 0-5: staging done
    first, last = arr.min(axis=1), arr.max(axis=1)
    lb = t[:, 5]                           # look-back done
    rel = t[:, 3]                          # barrier released
    ok = lb > 0
    def stat(x):
        x = x.astype(np.float64)
        return f"median {np.median(x):7.0f} ns  mean {x.mean():7.0f}  p90 {np.percentile(x, 90):7.0f}"
    print("  staging: first warp done -> last warp done      ", stat((last - first)[ok]))
    print("  look-back: first warp done -> base resolved     ", stat((lb - first)[ok]))
    print("  barrier release - last warp's staging           ", stat((rel - last)[ok]))
    print("  barrier release - look-back done                ", stat((rel - lb)[ok]))
    print(f"  tiles where the look-back ends after the last staging: {100.0 * np.mean((lb > last)[ok]):.1f}%")
    print("  wait of the average warp at that barrier        ", stat((rel[:, None] - arr)[ok].mean(axis=1)))


if __name__ == "__main__":
    main()
