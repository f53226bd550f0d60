import sys, ctypes, numpy as np
sys.path.insert(0, '.')
import paper_1902_08318_b200.jsontape as jtm
L = jtm.load_library(sys.argv[1])
import torch
from paper_1902_08318_b200 import Parser
from tools.gen import generate
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
d = generate(cfg, 64 << 20); n = len(d)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
p = Parser(); p.set_stream(s.cuda_stream)
host = torch.frombuffer(bytearray(d), dtype=torch.uint8).pin_memory()
p.copy_in(host.data_ptr(), n)
nt = (n + 16383) // 16384
dbg = torch.zeros(nt * 8, dtype=torch.int64, device='cuda')
L.jt_dbg_set.argtypes = [ctypes.c_void_p]
fl = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
for it in range(3):
    L.jt_dbg_set(dbg.data_ptr()); fl.zero_(); torch.cuda.synchronize()
    p.parse_async(n); p.finish(); torch.cuda.synchronize()
t = dbg.cpu().numpy().reshape(nt, 8).astype(np.float64)
t0 = t[:, 0].min()
names = ['start','classified','utf8+scan (pre-LB1)','after LB1','pre-LB2','staged','copyout-start','end']
dur = np.diff(t, axis=1)
for k in range(7):
    print(f'{names[k]:>22} -> {names[k+1]:<22} median {np.median(dur[:,k]):8.0f} ns  mean {dur[:,k].mean():8.0f}  p90 {np.percentile(dur[:,k],90):8.0f}')
life = t[:, 7] - t[:, 0]
print('lifetime median', np.median(life), 'total span', t[:, 7].max() - t0, 'ns; tiles', nt)
starts = np.sort(t[:, 0] - t0)
print('start times: first 5', starts[:5], 'tile 444..448', starts[444:449])
