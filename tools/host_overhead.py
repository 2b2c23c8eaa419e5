"""Dev tool: host-side cost per C-ABI call (Python + ctypes + tensor-map encoding + launch)
vs device time, for a short GEMM (cfg3 out-proj at TP8 per GPU)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")
M, K, N = 16384, 1024, 8192
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
b = (torch.randn((K, N), device=dev, generator=g) / 64).to(torch.bfloat16)
c = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
for _ in range(5):
    tpf.gemm(a, b, c)
torch.cuda.synchronize()
n = 50
t0 = time.perf_counter()
for _ in range(n):
    tpf.gemm(a, b, c)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6 * (t1 - t0) / n:.1f} us/call, wall {1e6 * (t2 - t0) / n:.1f} us/call")
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
torch.cuda.synchronize()
e0.record()
tpf.gemm(a, b, c)
e1.record()
torch.cuda.synchronize()
print(f"single launch device time {1e3 * e0.elapsed_time(e1):.1f} us")
comm = tpf.Communicator.create(0, 1, 0)
x = a.view(1, M, K)
y = c.view(1, M, N)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    comm.gemm_rs(x, b, y)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"comm.gemm_rs host enqueue {1e6 * (t1 - t0) / n:.1f} us/call, wall {1e6 * (t2 - t0) / n:.1f} us/call")
