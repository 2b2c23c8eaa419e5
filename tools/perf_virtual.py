"""Per-GPU cost of one rank of a real TP group, at full-GPU scale (148 SMs), with virtual
peers (Communicator.virtual_group: a self-ring -- the peers alias this rank's heap, so each
send fills the slot this rank reads one step later and the step-to-step waits are real). It runs the real per-rank protocol instructions: wire reads and forwarding for AG,
wire stores and inbox adds for RS, flag traffic. Compared against the same kernels in
compute-only mode and against the plain T = 1 GEMM of the per-rank shape, this isolates the
protocol's on-GPU overhead. NVLink latency is what it cannot show.
    python tools/perf_virtual.py [out.json]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")


def loop(fn, n):
    """Device time per call over n back-to-back calls (the host runs ahead, so launch latency
    and host-side argument setup are hidden as they are in a real layer sequence)."""
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    fn()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def measure(comm, fn, gemm, rounds=7, n=20):
    for _ in range(3):
        fn()
        gemm()
    f, c, g = [], [], []
    for _ in range(rounds):
        f.append(loop(fn, n))
        comm.set_compute_only(True)
        c.append(loop(fn, n))
        comm.set_compute_only(False)
        g.append(loop(gemm, n))
    return statistics.median(f), statistics.median(c), statistics.median(g)


res = {}
shapes = []
for T in (2, 4, 8):
    shapes += [("cfg2", T, 8192, 4096, 28672, 14336, 4096), ("cfg3", T, 16384, 8192, 10240, 8192, 8192)]
for cfg, T, S, K_ag, N_ag, K_rs, N_rs in shapes:
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((1, S // T, K_ag), device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn((K_ag, N_ag // T), device=dev, generator=g) / 64).to(torch.bfloat16)
    y = torch.empty((1, S, N_ag // T), device=dev, dtype=torch.bfloat16)
    xr = torch.randn((1, S, K_rs // T), device=dev, generator=g).to(torch.bfloat16)
    wr = (torch.randn((K_rs // T, N_rs), device=dev, generator=g) / 64).to(torch.bfloat16)
    yr = torch.empty((1, S // T, N_rs), device=dev, dtype=torch.bfloat16)
    xg = torch.randn((S, K_ag), device=dev, generator=g).to(torch.bfloat16)  # the gathered A
    yg = torch.empty((S, N_ag // T), device=dev, dtype=torch.bfloat16)
    yrg = torch.empty((S, N_rs), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, K_ag, N_ag // T),
                                                 tpf.sym_bytes_rs(T, 1, S, K_rs // T, N_rs, 1, tpf.BF16)))
    fa, ca, ga = measure(comm, lambda: comm.ag_gemm(x, w, y), lambda: tpf.gemm(xg, w, yg))
    fr, cr, gr = measure(comm, lambda: comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=tpf.BF16),
                         lambda: tpf.gemm(xr[0], wr, yrg))
    comm.close()
    fl_ag, fl_rs = 2.0 * S * K_ag * N_ag / T, 2.0 * S * K_rs * N_rs / T
    key = f"{cfg}_TP{T}"
    res[key] = {
        "ag_gemm": {"fused_ms": round(fa, 4), "compute_only_ms": round(ca, 4), "t1_gemm_ms": round(ga, 4),
                    "fused_tflops": round(fl_ag / fa / 1e9, 1), "protocol_overhead_us": round(1e3 * (fa - ca), 1)},
        "gemm_rs": {"fused_ms": round(fr, 4), "compute_only_ms": round(cr, 4), "t1_gemm_ms": round(gr, 4),
                    "fused_tflops": round(fl_rs / fr / 1e9, 1), "protocol_overhead_us": round(1e3 * (fr - cr), 1)},
    }
    print(key, json.dumps(res[key]), flush=True)
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/virtual_tp.json"
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as f:
    json.dump({"note": __doc__.split("\n")[0], "configs": res}, f, indent=1)
