"""Quick GPU sanity run (dev tool): T=1 GEMM vs torch, emulated AG/RS vs the oracle."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
os.environ.setdefault("TPF_TIMEOUT_MS", "2000")

import numpy as np
import torch

import paper_2604_24013_b200 as tpf
from oracle_lib import Oracle

O = Oracle()
dev = torch.device("cuda:0")
torch.manual_seed(0)


def gemm_case(M, K, N, ints=False):
    if ints:
        a = torch.randint(0, 5, (M, K), device=dev).to(torch.bfloat16)
        b = torch.randint(-2, 2, (K, N), device=dev).to(torch.bfloat16)
    else:
        a = torch.randn(M, K, device=dev).to(torch.bfloat16)
        b = (torch.randn(K, N, device=dev) / K ** 0.5).to(torch.bfloat16)
    out = torch.empty(M, N, device=dev, dtype=torch.float32)
    tpf.gemm(a, b, out)
    torch.cuda.synchronize()
    ref = a.float() @ b.float()
    err = (out - ref).abs().max().item()
    scale = ref.abs().max().item()
    print(f"gemm M={M} K={K} N={N} ints={ints}: max_abs_err={err:.3e} scale={scale:.3e}", flush=True)
    return err, scale


def rs_case(T, kind, m, B, S, K, N, wire=tpf.F32):
    x_full = O.randint((B, S, K), 0, 5, 11)
    w_full = O.randint((K, N), -2, 2, 12)
    want = O.row_parallel(T, kind, m, x_full, w_full)
    kl = K // T
    xs = np.stack([x_full[:, :, r * kl:(r + 1) * kl] for r in range(T)])
    ws = np.stack([w_full[r * kl:(r + 1) * kl] for r in range(T)])
    x = torch.tensor(xs, dtype=torch.bfloat16, device=dev).contiguous()
    w = torch.tensor(ws, dtype=torch.bfloat16, device=dev).contiguous()
    out = torch.full((T, B, S // T, N), float("nan"), device=dev, dtype=torch.float32)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_rs(T, B, S, kl, N, m, wire))
    comm.gemm_rs(x, w, out, kind=kind, m=m, wire=wire)
    comm.sync()
    got = out.cpu().numpy().astype(np.float64)
    err = np.abs(got - want).max()
    print(f"rs T={T} kind={kind} m={m} B={B} S={S} K={K} N={N}: max_abs_err={err}", flush=True)
    comm.close()
    return err


def ag_case(T, m, B, S, K, N):
    x_full = O.randint((B, S, K), 0, 5, 21)
    w_full = O.randint((K, N), -2, 2, 22)
    want = O.column_parallel(T, m, x_full, w_full)
    sl, nl = S // T, N // T
    xs = np.stack([x_full[:, r * sl:(r + 1) * sl] for r in range(T)])
    ws = np.stack([w_full[:, r * nl:(r + 1) * nl] for r in range(T)])
    x = torch.tensor(xs, dtype=torch.bfloat16, device=dev).contiguous()
    w = torch.tensor(ws, dtype=torch.bfloat16, device=dev).contiguous()
    out = torch.full((T, B, S, nl), float("nan"), device=dev, dtype=torch.float32)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ag(T, B, S, K, nl, m))
    comm.ag_gemm(x, w, out, m=m)
    comm.sync()
    got = out.cpu().numpy().astype(np.float64)
    err = np.abs(got - want).max()
    print(f"ag T={T} m={m} B={B} S={S} K={K} N={N}: max_abs_err={err}", flush=True)
    comm.close()
    return err


def bench_gemm(M, K, N, iters=20):
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    b = (torch.randn(K, N, device=dev) / K ** 0.5).to(torch.bfloat16)
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        tpf.gemm(a, b, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        tpf.gemm(a, b, out)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / iters
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    tc = e0.elapsed_time(e1) / iters
    fl = 2 * M * K * N
    print(f"bench gemm {M}x{K}x{N}: tpf {t*1e3:.1f} us {fl/t/1e9:.1f} TF/s | cublas {tc*1e3:.1f} us {fl/tc/1e9:.1f} TF/s", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    print("sms", tpf.lib().tpf_device_sms(), flush=True)
    if which in ("gemm", "all"):
        gemm_case(128, 64, 256, ints=True)
        gemm_case(256, 256, 512, ints=True)
        gemm_case(1024, 1024, 1024)
        gemm_case(300, 200, 136, ints=True)
        gemm_case(2048, 4096, 3584)
    if which in ("rs", "all"):
        rs_case(2, 0, 1, 1, 256, 128, 256)
        rs_case(4, 0, 1, 2, 64, 32, 32)
        rs_case(4, 1, 1, 2, 512, 256, 512)
        rs_case(4, 2, 1, 2, 512, 256, 512)
        rs_case(8, 0, 2, 2, 64, 64, 32)
    if which in ("ag", "all"):
        ag_case(2, 1, 1, 256, 128, 256)
        ag_case(4, 1, 2, 64, 32, 64)
        ag_case(4, 2, 2, 512, 256, 512)
        ag_case(8, 2, 2, 64, 32, 64)
    if which in ("bench", "all"):
        bench_gemm(8192, 4096, 8192)
        bench_gemm(8192, 4096, 28672)
        bench_gemm(8192, 14336, 4096)
