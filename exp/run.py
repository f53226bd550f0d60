import sys, json, os, ctypes
sys.path.insert(0, '.')
import paper_1902_08318_b200.jsontape as jtm
jtm.load_library(sys.argv[1])
import torch
from paper_1902_08318_b200 import Parser
from tools.gen import generate
d = generate(1, 64 << 20); n = len(d)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
p = Parser(); p.set_stream(s.cuda_stream)
host = torch.frombuffer(bytearray(d), dtype=torch.uint8).pin_memory()
p.copy_in(host.data_ptr(), n)
p.profile(True)
fl = torch.empty(256 << 20, dtype=torch.uint8, device='cuda')
ts = []
for i in range(8):
    fl.zero_(); p.parse_async(n); p.finish(); ts.append(p.kernel_times()['stage1'])
print(sys.argv[1], 'stage1 ms', sorted(ts)[len(ts)//2])
