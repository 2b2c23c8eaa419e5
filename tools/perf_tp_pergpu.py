"""Per-GPU GEMM shapes of real TP = 2/4/8 (cfg2 / cfg3) on the full 148-SM GPU: the T = 1
kernel over one rank's operands measures what each GPU computes, including wave
quantization (tiles per launch vs 74 CTA pairs). cuBLAS on the same shapes for reference."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")


def t_ms(fn, n=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


shapes = []
for T in (1, 2, 4, 8):
    shapes.append((f"cfg2 AG gate||up TP{T}", 8192, 4096, 28672 // T))
    shapes.append((f"cfg2 RS down TP{T}", 8192, 14336 // T, 4096))
for T in (2, 4, 8):
    shapes.append((f"cfg3 AG qkv TP{T}", 16384, 8192, 10240 // T))
    shapes.append((f"cfg3 RS out TP{T}", 16384, 8192 // T, 8192))
for name, M, K, N in shapes:
    g = torch.Generator(device=dev).manual_seed(0)
    a = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
    b = (torch.randn((K, N), device=dev, generator=g) / 64).to(torch.bfloat16)
    c = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
    ours = t_ms(lambda: tpf.gemm(a, b, c))
    cub = t_ms(lambda: torch.matmul(a, b, out=c))
    tiles = (M // 256) * ((N + 255) // 256)
    fl = 2.0 * M * K * N
    print(f"{name:24s} M={M} K={K} N={N}: tiles={tiles} waves={tiles / 74:.2f}  ours {fl / ours / 1e9:7.0f} TF/s"
          f"  cuBLAS {fl / cub / 1e9:7.0f} TF/s", flush=True)
