"""Dev tool: one T = 1 GEMM of the given shape for an ncu capture of the fused kernel.
    ncu --set full -k regex:tpf_fused -c 1 python tools/ncu_gemm.py M K N"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

M, K, N = (int(v) for v in sys.argv[1:4])
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
a = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
b = (torch.randn((K, N), device=dev, generator=g) / 64).to(torch.bfloat16)
c = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
tpf.gemm(a, b, c)
torch.cuda.synchronize()
print("ok")
