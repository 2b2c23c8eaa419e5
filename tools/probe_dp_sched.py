"""Dev probe: per-GPU cfg4 DP gradient RS (virtual peers, TP = 8 ranks) for each schedule against
the plain T = 1 GEMM of the same shapes.   python tools/probe_dp_sched.py"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")


def loop(fn, n=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / n


T, M, K, N = 8, 4096, 2048, 8192
g = torch.Generator(device=dev).manual_seed(1)
X = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
dY = (torch.randn((M, N), device=dev, generator=g) / 64).to(torch.bfloat16)
dW = torch.empty((K // T, N), device=dev, dtype=torch.bfloat16)
dWf = torch.empty((K, N), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.virtual_group(T, tpf.sym_bytes_rs(T, 1, K, M, N, 1, tpf.BF16))
one = tpf.Communicator.create(0, 1, 0)
for rnd in range(3):
    res = {"plain": loop(lambda: one.dp_grad_rs(X, dY, dWf))}
    for name, kind in (("ring", tpf.RING), ("circular", tpf.CIRCULAR), ("pairwise", tpf.PAIRWISE)):
        res[name] = loop(lambda: comm.dp_grad_rs(X, dY, dW, kind=kind, wire=tpf.BF16))
    print(" ".join(f"{k} {v:6.1f}" for k, v in res.items()), flush=True)
comm.sync()
comm.close()
one.close()
