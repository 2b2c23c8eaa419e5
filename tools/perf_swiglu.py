"""Dev tool: AG-GEMM gate||up with and without the fused SwiGLU epilogue, T = 1..8 (local group)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")
S, D, F = 8192, 4096, 14336


def t_ms(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for T in (1, 2, 4, 8):
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((T, 1, S // T, D), device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn((T, D, 2 * F // T), device=dev, generator=g) / 64).to(torch.bfloat16)
    o_full = torch.empty((T, 1, S, 2 * F // T), device=dev, dtype=torch.bfloat16)
    o_half = torch.empty((T, 1, S, F // T), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ag(T, 1, S, D, 2 * F // T, 1))
    r = {}
    for co in (False, True):
        comm.set_compute_only(co)
        r[("none", co)] = t_ms(lambda: comm.ag_gemm(x, w, o_full))
        r[("swiglu", co)] = t_ms(lambda: comm.ag_gemm(x, w, o_half, act=tpf.ACT_SWIGLU))
    comm.set_compute_only(False)
    comm.sync()
    comm.close()
    print(f"T={T}: plain {r[('none', False)]:.3f} (co {r[('none', True)]:.3f})  "
          f"swiglu {r[('swiglu', False)]:.3f} (co {r[('swiglu', True)]:.3f}) ms", flush=True)
