"""PCIe probe: H2D / D2H / both at once for copy sizes 1-64 MiB (pinned host memory).

    python tools/pcie_probe.py   (on the GPU box)
"""
import torch, time
N = 64 << 20
h_in = torch.empty(N, dtype=torch.uint8).pin_memory()
h_out = torch.empty(N, dtype=torch.uint8).pin_memory()
d_in = torch.empty(N, dtype=torch.uint8, device="cuda")
d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(ch_up, ch_dn, both=True, up=True):
    torch.cuda.synchronize()
    t = time.perf_counter()
    if up:
        with torch.cuda.stream(s1):
            for o in range(0, N, ch_up):
                d_in[o:o + ch_up].copy_(h_in[o:o + ch_up], non_blocking=True)
    if both:
        with torch.cuda.stream(s2):
            for o in range(0, N, ch_dn):
                h_out[o:o + ch_dn].copy_(d_out[o:o + ch_dn], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3
for _ in range(3): run(4 << 20, 2 << 20)
for ch in (1 << 20, 2 << 20, 4 << 20, 16 << 20, 64 << 20):
    a = min(run(ch, ch, both=False) for _ in range(5))
    b = min(run(ch, ch, both=True, up=False) for _ in range(5))
    c = min(run(ch, ch, both=True) for _ in range(5))
    print(f"chunk {ch>>20} MiB: H2D alone {a:.3f} ms ({N/a/1e6:.1f} GB/s), D2H alone {b:.3f} ms ({N/b/1e6:.1f}), both {c:.3f} ms ({2*N/c/1e6:.1f} GB/s aggregate)")
