"""Dev tool: time the fused ops on one GPU (local group = all T ranks in one launch),
fused vs compute-only (same kernel, no flag waits / wire traffic).

    python tools/perf_fused.py [cfg2|cfg3] [T ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")
stream = torch.cuda.current_stream()


def timeit(fn, n=10, warm=3, reps=3):
    """min over `reps` batches of the mean of n back-to-back calls (us)."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / n * 1e3)
    return best


def run(T, S, K_ag, N_ag, K_rs, N_rs, wire=tpf.BF16, kinds=(tpf.RING,)):
    g = torch.Generator(device=dev).manual_seed(0)
    sl = S // T
    x = torch.randn((T, 1, sl, K_ag), device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn((T, K_ag, N_ag // T), device=dev, generator=g) / 64).to(torch.bfloat16)
    out = torch.empty((T, 1, S, N_ag // T), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.local_group(T, max(tpf.sym_bytes_ag(T, 1, S, K_ag, N_ag // T, 1),
                                               tpf.sym_bytes_rs(T, 1, S, K_rs // T, N_rs, 1, tpf.F32)))
    flops_ag = 2.0 * S * K_ag * N_ag
    f = timeit(lambda: comm.ag_gemm(x, w, out))
    comm.set_compute_only(True)
    c = timeit(lambda: comm.ag_gemm(x, w, out))
    comm.set_compute_only(False)
    comm.sync()
    print(f"T={T} AG  S={S} K={K_ag} N={N_ag}: fused {f:8.1f} us ({flops_ag / f / 1e6:6.0f} TF/s)  "
          f"compute-only {c:8.1f} us  exposed {f - c:7.1f} us", flush=True)
    xr = torch.randn((T, 1, S, K_rs // T), device=dev, generator=g).to(torch.bfloat16)
    wr = (torch.randn((T, K_rs // T, N_rs), device=dev, generator=g) / 64).to(torch.bfloat16)
    o = torch.empty((T, 1, sl, N_rs), device=dev, dtype=torch.bfloat16)
    flops_rs = 2.0 * S * K_rs * N_rs
    for kind in kinds:
        for wd in ((wire,) if wire is not None else (tpf.BF16, tpf.F32)):
            f = timeit(lambda: comm.gemm_rs(xr, wr, o, kind=kind, wire=wd))
            comm.set_compute_only(True)
            c = timeit(lambda: comm.gemm_rs(xr, wr, o, kind=kind, wire=wd))
            comm.set_compute_only(False)
            comm.sync()
            print(f"T={T} RS  S={S} K={K_rs} N={N_rs} {tpf.KIND_NAMES[kind]:>9} wire={'bf16' if wd == tpf.BF16 else 'f32 '}: "
                  f"fused {f:8.1f} us ({flops_rs / f / 1e6:6.0f} TF/s)  compute-only {c:8.1f} us  exposed {f - c:7.1f} us",
                  flush=True)
    comm.close()


if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    Ts = [int(v) for v in sys.argv[2:]] or [1, 2, 4, 8]
    for T in Ts:
        if cfg == "cfg2":   # Llama-3-8B MLP: gate||up (4096 -> 28672), down (14336 -> 4096), S=8192
            run(T, 8192, 4096, 28672, 14336, 4096, wire=None,
                kinds=(tpf.RING, tpf.PAIRWISE, tpf.CIRCULAR) if T > 1 else (tpf.RING,))
        else:               # Llama-3-70B attn: QKV (8192 -> 10240), out-proj (8192 -> 8192), S=16384
            run(T, 16384, 8192, 10240, 8192, 8192)
