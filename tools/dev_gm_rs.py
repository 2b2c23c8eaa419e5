"""Dev tool: T = 1 GEMM time of the cfg2 down projection (8192 x 14336 x 4096) and the gate||up
projection for the current TPF_GROUP_M."""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
res = []
for M, K, N in ((8192, 14336, 4096), (8192, 4096, 28672)):
    a = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
    b = (torch.randn((K, N), device=dev, generator=g) / 64).to(torch.bfloat16)
    c = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
    for _ in range(5):
        tpf.gemm(a, b, c)
    ts = []
    for _ in range(9):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        torch.cuda.synchronize()
        e0.record()
        tpf.gemm(a, b, c)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res.append(2.0 * M * K * N / statistics.median(ts) / 1e9)
print(os.environ.get("TPF_GROUP_M", "16"), "RS-shape %.0f TF/s  AG-shape %.0f TF/s" % tuple(res))
