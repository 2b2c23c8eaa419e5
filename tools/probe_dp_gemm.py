"""Dev probe: the DP-gradient GEMM (MN-major A = X^T read from row-major X, MODE_DP_GRAD) against a
K-major GEMM of the same size (T = 1 instances), to separate the operand layout from tile
quantization.   python tools/probe_dp_gemm.py"""
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


one = tpf.Communicator.create(0, 1, 0)
for M, K, N in ((4096, 2048, 8192), (8192, 2048, 8192), (4096, 4096, 8192)):
    g = torch.Generator(device=dev).manual_seed(0)
    X = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)      # tokens x features
    dY = torch.randn((M, N), device=dev, generator=g).to(torch.bfloat16)
    dW = torch.empty((K, N), device=dev, dtype=torch.bfloat16)
    XT = X.t().contiguous()                                                   # K-major copy
    out = torch.empty((K, N), device=dev, dtype=torch.bfloat16)
    t_dp = loop(lambda: one.dp_grad_rs(X, dY, dW))
    t_km = loop(lambda: tpf.gemm(XT, dY, out))
    fl = 2.0 * M * K * N
    print(f"dW[{K}x{N}] over {M} tokens: MN-major A {t_dp:7.1f} us ({fl / t_dp / 1e6:6.0f} TF/s) | "
          f"K-major A {t_km:7.1f} us ({fl / t_km / 1e6:6.0f} TF/s)")
one.close()
