"""Dev tool: per-GPU TP = 8 fused ops (virtual peers, cfg2) timed three ways -- back-to-back
eager calls between two events (the bench's method), the same 20 calls replayed from a CUDA
graph (no host work), and the host enqueue time per eager call -- to tell host-bound loops
from device time.  python tools/loop_vs_graph.py"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

T, S, D, F = 8, 8192, 4096, 14336
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn((1, S // T, D), device=dev, generator=g).to(torch.bfloat16)
w = (torch.randn((D, 2 * F // T), device=dev, generator=g) / 64).to(torch.bfloat16)
act = torch.empty((1, S, F // T), device=dev, dtype=torch.bfloat16)
wd = (torch.randn((F // T, D), device=dev, generator=g) / 64).to(torch.bfloat16)
y = torch.empty((1, S // T, D), device=dev, dtype=torch.bfloat16)
xg = torch.randn((1, S, D), device=dev, generator=g).to(torch.bfloat16)
yg = torch.empty((1, S, D), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, D, 2 * F // T), tpf.sym_bytes_rs(T, 1, S, F // T, D, 1, tpf.BF16)))
one = tpf.Communicator.create(0, 1, 0)
s = torch.cuda.Stream()
ops = {
    "ag": lambda: comm.ag_gemm(x, w, act, act=tpf.ACT_SWIGLU, stream=s),
    "rs": lambda: comm.gemm_rs(act, wd, y, kind=tpf.RING, wire=tpf.BF16, stream=s),
    "plain_ag": lambda: one.ag_gemm(xg, w, act, act=tpf.ACT_SWIGLU, stream=s),
    "plain_rs": lambda: one.gemm_rs(act, wd, yg, stream=s),
}
n = 20
for name, fn in ops.items():
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    s.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    h0 = time.perf_counter()
    e0.record(s)
    for _ in range(n):
        fn()
    h1 = time.perf_counter()
    e1.record(s)
    s.synchronize()
    loop = 1e3 * e0.elapsed_time(e1) / n
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for _ in range(n):
            fn()
    res = []
    with torch.cuda.stream(s):  # replay() launches on the current stream
        graph.replay()
        s.synchronize()
        for _ in range(3):
            e0.record(s)
            graph.replay()
            e1.record(s)
            s.synchronize()
            res.append(1e3 * e0.elapsed_time(e1) / n)
    print(f"{name:9s} eager loop {loop:7.1f} us/call   graph {min(res):7.1f} us/call   host enqueue "
          f"{1e6 * (h1 - h0) / n:6.1f} us/call", flush=True)
comm.sync(s)
