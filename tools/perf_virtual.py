"""Per-GPU cost of one rank of a real TP / DP group at full-GPU scale (148 SMs), with virtual
peers (Communicator.virtual_group: a self-ring -- the peers alias this rank's heap, so each send
fills the slot this rank reads one step later and the step-to-step waits are real). It runs the
real per-rank protocol instructions (wire reads and forwarding for AG, wire stores and inbox adds
for RS, flags), against the plain T = 1 GEMM of the same per-rank shapes: exposed = fused - plain,
and t_roof = max(FLOPs at the measured bf16 burst peak, wire bytes over NVLink) at 900 GB/s
(north_star) and at the measured 770 GB/s peer copy. NVLink latency / bandwidth is what it cannot
show. Medians of 7 rounds of 20 back-to-back calls, fused and plain alternating; TP = 8 first.
    python tools/perf_virtual.py [out.json]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")
PEAK = 1638.5e12
try:
    PEAK = json.load(open(os.path.join(os.getcwd(), "MEASURED_PEAKS.json")))["bf16_tflops"] * 1e12
except Exception:
    pass


def loop(fn, n):
    """Device time per call over n back-to-back calls (the host runs ahead)."""
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    fn()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def measure(fn, plain, rounds=7, n=20):
    for _ in range(3):
        fn()
        plain()
    f, g = [], []
    for _ in range(rounds):
        f.append(loop(fn, n))
        g.append(loop(plain, n))
    return statistics.median(f), statistics.median(g)


def row(fused_ms, plain_ms, flops, wire_bytes):
    r900 = max(flops / PEAK, wire_bytes / 900e9) * 1e3
    r770 = max(flops / PEAK, wire_bytes / 770e9) * 1e3
    return {"fused_ms": round(fused_ms, 4), "plain_gemm_ms": round(plain_ms, 4),
            "fused_over_plain": round(fused_ms / plain_ms, 3), "exposed_us": round(1e3 * (fused_ms - plain_ms), 1),
            "fused_tflops": round(flops / fused_ms / 1e9, 1), "t_roof_ms": round(r900, 4),
            "frac_of_t_roof": round(r900 / fused_ms, 3), "frac_of_t_roof_link770": round(r770 / fused_ms, 3)}


res = {}
one = tpf.Communicator.create(0, 1, 0)
for T in (8, 4, 2):
    for cfg, S, K_ag, N_ag, K_rs, N_rs in (("cfg2", 8192, 4096, 28672, 14336, 4096),
                                           ("cfg3", 16384, 8192, 10240, 8192, 8192)):
        g = torch.Generator(device=dev).manual_seed(0)
        x = torch.randn((1, S // T, K_ag), device=dev, generator=g).to(torch.bfloat16)
        w = (torch.randn((K_ag, N_ag // T), device=dev, generator=g) / 64).to(torch.bfloat16)
        y = torch.empty((1, S, N_ag // T), device=dev, dtype=torch.bfloat16)
        xr = torch.randn((1, S, K_rs // T), device=dev, generator=g).to(torch.bfloat16)
        wr = (torch.randn((K_rs // T, N_rs), device=dev, generator=g) / 64).to(torch.bfloat16)
        yr = torch.empty((1, S // T, N_rs), device=dev, dtype=torch.bfloat16)
        xg = torch.randn((1, S, K_ag), device=dev, generator=g).to(torch.bfloat16)  # the gathered A
        yrg = torch.empty((1, S, N_rs), device=dev, dtype=torch.bfloat16)
        comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, K_ag, N_ag // T),
                                                     tpf.sym_bytes_rs(T, 1, S, K_rs // T, N_rs, 1, tpf.BF16)))
        fa, ga = measure(lambda: comm.ag_gemm(x, w, y), lambda: one.ag_gemm(xg, w, y))
        fr, gr = measure(lambda: comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=tpf.BF16),
                         lambda: one.gemm_rs(xr, wr, yrg))
        comm.sync()
        comm.close()
        moved = (T - 1) / T * S * 2
        key = f"{cfg}_TP{T}"
        res[key] = {"ag_gemm": row(fa, ga, 2.0 * S * K_ag * N_ag / T, moved * K_ag),
                    "gemm_rs_bf16_wire": row(fr, gr, 2.0 * S * K_rs * N_rs / T, moved * N_rs)}
        print(key, json.dumps(res[key]), flush=True)
    if T == 8:
        # cfg4 DP (8 ranks, 4096 tokens / rank, a 2048 x 8192 weight): gradient RS of dW and
        # parameter AG fused into the forward GEMM
        M, K, N = 4096, 2048, 8192
        g = torch.Generator(device=dev).manual_seed(1)
        X = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
        dY = (torch.randn((M, N), device=dev, generator=g) / 64).to(torch.bfloat16)
        dW = torch.empty((K // T, N), device=dev, dtype=torch.bfloat16)
        dWf = torch.empty((K, N), device=dev, dtype=torch.bfloat16)
        Wr = (torch.randn((N // T, K), device=dev, generator=g) / 45).to(torch.bfloat16)
        Wf = (torch.randn((N, K), device=dev, generator=g) / 45).to(torch.bfloat16)
        out = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_rs(T, 1, K, M, N, 1, tpf.BF16),
                                                     tpf.sym_bytes_dp_ag(T, K, N // T)))
        fd, gd = measure(lambda: comm.dp_grad_rs(X, dY, dW, kind=tpf.RING, wire=tpf.BF16),
                         lambda: one.dp_grad_rs(X, dY, dWf))
        fp, gp = measure(lambda: comm.dp_param_ag_gemm(X, Wr, out), lambda: one.dp_param_ag_gemm(X, Wf, out))
        comm.sync()
        comm.close()
        wire = (T - 1) / T * K * N * 2
        res["cfg4_DP8"] = {"dp_grad_rs_bf16_wire": row(fd, gd, 2.0 * M * K * N, wire),
                           "dp_param_ag_gemm": row(fp, gp, 2.0 * M * K * N, wire)}
        print("cfg4_DP8", json.dumps(res["cfg4_DP8"]), flush=True)
one.close()
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/virtual_tp.json"
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
with open(out, "w") as f:
    json.dump({"note": " ".join(__doc__.split("\n")[:2]), "peak_tflops": PEAK / 1e12, "configs": res}, f, indent=1)
