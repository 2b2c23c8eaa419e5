"""Dev tool: per-call device time vs. call-to-call interval for back-to-back per-GPU fused calls
(virtual peers) and the plain GEMM, to separate kernel duration from gaps between kernels.
    python tools/loop_gaps.py [T]"""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2
S, K, N = 8192, 4096, 28672
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn((1, S // T, K), device=dev, generator=g).to(torch.bfloat16)
xg = torch.randn((1, S, K), device=dev, generator=g).to(torch.bfloat16)
w = (torch.randn((K, N // T), device=dev, generator=g) / 64).to(torch.bfloat16)
y = torch.empty((1, S, N // T), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.virtual_group(T, tpf.sym_bytes_ag(T, 1, S, K, N // T))
one = tpf.Communicator.create(0, 1, 0)
for name, fn in (("fused", lambda: comm.ag_gemm(x, w, y)), ("plain", lambda: one.ag_gemm(xg, w, y)),
                 ("fused", lambda: comm.ag_gemm(x, w, y)), ("plain", lambda: one.ag_gemm(xg, w, y))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    n = 20
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * n)]
    for i in range(n):
        ev[2 * i].record()
        fn()
        ev[2 * i + 1].record()
    torch.cuda.synchronize()
    dur = [ev[2 * i].elapsed_time(ev[2 * i + 1]) * 1e3 for i in range(n)]
    per = ev[0].elapsed_time(ev[-1]) * 1e3 / n
    print(f"T={T} {name}: per call {per:.1f} us, kernel (event pair) median {statistics.median(dur):.1f} "
          f"min {min(dur):.1f} max {max(dur):.1f} us", flush=True)
comm.sync()
