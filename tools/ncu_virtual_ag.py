"""Dev tool: one per-GPU AG-GEMM of a TP group (virtual peers) and the plain GEMM of the same
per-rank work, for an ncu comparison. python tools/ncu_virtual_ag.py T [compute_only]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

T = int(sys.argv[1])
co = len(sys.argv) > 2 and sys.argv[2] == "1"
S, K, N = 8192, 4096, 28672
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn((1, S // T, K), device=dev, generator=g).to(torch.bfloat16)
w = (torch.randn((K, N // T), device=dev, generator=g) / 64).to(torch.bfloat16)
y = torch.empty((1, S, N // T), device=dev, dtype=torch.bfloat16)
xg = torch.randn((S, K), device=dev, generator=g).to(torch.bfloat16)
yg = torch.empty((S, N // T), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.virtual_group(T, tpf.sym_bytes_ag(T, 1, S, K, N // T))
comm.set_compute_only(co)
comm.ag_gemm(x, w, y)
tpf.gemm(xg, w, yg)
torch.cuda.synchronize()
comm.close()
print("ok")
