"""Dev tool: kernel durations and the idle gap between back-to-back launches (CUPTI via
torch.profiler), for the per-GPU TP8 shapes: what a launch + prologue costs between two
fused calls on one stream.  python tools/launch_gaps.py"""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")
T, S = 8, 8192
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn((1, S // T, 4096), device=dev, generator=g).to(torch.bfloat16)
w = (torch.randn((4096, 28672 // T), device=dev, generator=g) / 64).to(torch.bfloat16)
y = torch.empty((1, S, 28672 // T), device=dev, dtype=torch.bfloat16)
xr = torch.randn((1, S, 14336 // T), device=dev, generator=g).to(torch.bfloat16)
wr = (torch.randn((14336 // T, 4096), device=dev, generator=g) / 64).to(torch.bfloat16)
yr = torch.empty((1, S // T, 4096), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, 4096, 28672 // T),
                                             tpf.sym_bytes_rs(T, 1, S, 14336 // T, 4096, 1, tpf.BF16)))


def run(name, fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        torch.cuda._sleep(5_000_000)
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
    ks = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
                 and "tpf_" in e.name], key=lambda e: e.time_range.start)
    dur = [e.time_range.end - e.time_range.start for e in ks]
    gaps = [b.time_range.start - a.time_range.end for a, b in zip(ks, ks[1:])]
    per = (ks[-1].time_range.end - ks[0].time_range.start) / len(ks)
    print(f"{name}: {len(ks)} kernels, duration median {statistics.median(dur):.1f} us, gap median "
          f"{statistics.median(gaps):.2f} us (min {min(gaps):.2f} max {max(gaps):.2f}), per call {per:.1f} us", flush=True)


run("AG  TP8 fused", lambda: comm.ag_gemm(x, w, y))
run("RS  TP8 fused", lambda: comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=tpf.BF16))
run("AG+RS alternating", lambda: (comm.ag_gemm(x, w, y), comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=tpf.BF16)))
yg = torch.empty((S, 4096), device=dev, dtype=torch.bfloat16)
run("GEMM 8192x1792x4096", lambda: tpf.gemm(xr[0], wr, yg))
comm.close()
