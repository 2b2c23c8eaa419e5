"""Measure every BASELINE.json config on one B200 (dev / evidence tool).

T = 1 runs the real single-GPU path. T > 1 runs the single-GPU local group: all T ranks
in one launch, each on 148/T SMs, wire traffic through local HBM rather than NVLink.
For each fused op it reports time, TFLOP/s, and exposed comm = fused - compute-only
(the same kernel with flag waits and wire traffic disabled).

    python tools/perf_configs.py [out.json]
"""
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_24013_b200 as tpf

DEV = torch.device("cuda:0")


def timeit(fn, n=5, warm=2, reps=3):
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
        best = min(best, e0.elapsed_time(e1) / n)
    return best  # ms


def _one(fn):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def fused_and_exposed(comm, fn, flops, rounds=7):
    """Single calls, fused and compute-only ALTERNATING (so power-cap clock drift lands on
    both equally); medians. Back-to-back timing swings by 10-20% on these boxes as the
    power cap engages, which swamps the effect being measured."""
    for _ in range(2):
        fn()
    fused, co = [], []
    for _ in range(rounds):
        fused.append(_one(fn))
        if comm.world > 1:
            comm.set_compute_only(True)
            co.append(_one(fn))
            comm.set_compute_only(False)
    comm.sync()
    t = statistics.median(fused)
    c = statistics.median(co) if co else t
    return {"ms": round(t, 4), "tflops": round(flops / (t * 1e-3) / 1e12, 1),
            "compute_only_ms": round(c, 4), "exposed_us": round(1e3 * (t - c), 1)}


def rnd(shape, scale=1.0, seed=0):
    g = torch.Generator(device=DEV).manual_seed(seed)
    return (torch.randn(shape, device=DEV, generator=g) * scale).to(torch.bfloat16)


def ag_rs(T, S, K_ag, N_ag, K_rs, N_rs, wire=tpf.BF16, out_f32=False):
    od = torch.float32 if out_f32 else torch.bfloat16
    x = rnd((T, 1, S // T, K_ag), 1.0, 1)
    w = rnd((T, K_ag, N_ag // T), K_ag ** -0.5, 2)
    y = torch.empty((T, 1, S, N_ag // T), device=DEV, dtype=od)
    xr = rnd((T, 1, S, K_rs // T), 1.0, 3)
    wr = rnd((T, K_rs // T, N_rs), K_rs ** -0.5, 4)
    yr = torch.empty((T, 1, S // T, N_rs), device=DEV, dtype=od)
    comm = tpf.Communicator.local_group(T, max(tpf.sym_bytes_ag(T, 1, S, K_ag, N_ag // T),
                                               tpf.sym_bytes_rs(T, 1, S, K_rs // T, N_rs, 1, wire)))
    res = {"ag_gemm": fused_and_exposed(comm, lambda: comm.ag_gemm(x, w, y), 2.0 * S * K_ag * N_ag),
           "gemm_rs": fused_and_exposed(comm, lambda: comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=wire),
                                        2.0 * S * K_rs * N_rs)}
    comm.close()
    return res


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/configs.json"
    res = {"note": "T=1: single-GPU path. T>1: single-GPU local group (T ranks in one launch, 148/T SMs each, "
                   "wire via local HBM, not NVLink). exposed_us = fused - compute-only, medians of single calls "
                   "with fused / compute-only alternating.", "configs": {}}
    C = res["configs"]
    # cfg1: CPU-reference config (T=4, M=K=N=4096), fp32 wire / output as the parity config
    C["cfg1_T4_4096cubed_fp32"] = ag_rs(4, 4096, 4096, 4096, 4096, 4096, wire=tpf.F32, out_f32=True)
    # cfg2: Llama-3-8B MLP (gate||up 4096 -> 28672, down 14336 -> 4096), S = 8192
    for T in (1, 2, 4, 8):
        C[f"cfg2_llama3_8b_mlp_T{T}"] = ag_rs(T, 8192, 4096, 28672, 14336, 4096)
    # cfg3: Llama-3-70B attention projections, S = 16384 (QKV 8192 -> 10240, out 8192 -> 8192)
    for T in (1, 2, 4, 8):
        C[f"cfg3_llama3_70b_attn_proj_T{T}"] = ag_rs(T, 16384, 8192, 10240, 8192, 8192)
    # cfg4: DP (8 ranks), Llama-3.2-1B-class MLP weight 2048 x 8192, 4096 tokens per rank
    T, M, K, N = 8, 4096, 2048, 8192
    X = rnd((T, M, K), 1.0, 5)
    dY = rnd((T, M, N), 0.02, 6)
    dW = torch.empty((T, K // T, N), device=DEV)
    W = rnd((N, K), K ** -0.5, 7)
    Wr = W.reshape(T, N // T, K).contiguous()
    Yp = torch.empty((T, M, N), device=DEV, dtype=torch.bfloat16)
    comm = tpf.Communicator.local_group(T, max(tpf.sym_bytes_rs(T, 1, K, M, N, 1, tpf.BF16),
                                               tpf.sym_bytes_dp_ag(T, K, N // T)))
    C["cfg4_dp_T8_grad_rs"] = fused_and_exposed(
        comm, lambda: comm.dp_grad_rs(X, dY, dW, kind=tpf.RING, wire=tpf.BF16), 2.0 * T * M * K * N)
    C["cfg4_dp_T8_param_ag"] = fused_and_exposed(comm, lambda: comm.dp_param_ag_gemm(X, Wr, Yp),
                                                 2.0 * T * M * K * N)
    comm.close()
    # cfg5: UP on a Llama-3-8B layer (4 q heads x 128 per rank at T=8), S = 32768
    T, heads, S, Dh = 8, 4, 32768, 128
    q, k, v = (rnd((T, heads, S, Dh), 1.0, 10 + i) for i in range(3))
    o = torch.empty((T, 1, S // T, T * heads * Dh), device=DEV, dtype=torch.bfloat16)
    comm = tpf.Communicator.local_group(T, 1 << 27)
    flops = 4.0 * T * heads * S * S * Dh  # whole group: QK^T + PV, non-causal
    t = timeit(lambda: comm.attention_a2a(q, k, v, o, 1, heads), n=2, warm=2, reps=3)
    comm.sync()
    comm.close()
    C["cfg5_up_T8_S32768"] = {"ms": round(t, 3), "tflops": round(flops / (t * 1e-3) / 1e12, 1),
                              "note": "one persistent tcgen05 flash-attention launch (two query tiles per CTA, S/P/O in "
                                      "TMEM) whose epilogue pushes O tiles to the slice owner + flags"}
    # cfg5 end to end: sequence-sharded q/k/v -> first all-to-all -> fused attention -> output a2a
    H = T * heads
    qs, ks, vs = (rnd((T, H, S // T, Dh), 1.0, 20 + i) for i in range(3))
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ulysses(T, 1, H, S, Dh))
    t_full = timeit(lambda: comm.ulysses_attention(qs, ks, vs, o, 1, H), n=2, warm=2, reps=3)
    hq, hk, hv = (torch.empty((T, heads, S, Dh), device=DEV, dtype=torch.bfloat16) for _ in range(3))
    t_a2a = timeit(lambda: comm.ulysses_a2a(qs, ks, vs, hq, hk, hv, 1, H), n=3, warm=1, reps=3)
    comm.sync()
    comm.close()
    a2a_bytes = 3 * T * H * (S // T) * Dh * 2  # every element read once and written once
    C["cfg5_up_T8_S32768_end_to_end"] = {
        "ms": round(t_full, 3), "tflops": round(flops / (t_full * 1e-3) / 1e12, 1),
        "first_a2a_standalone_ms": round(t_a2a, 3),
        "first_a2a_GBps_per_direction": round(a2a_bytes / (t_a2a * 1e-3) / 1e9, 1),
        "note": "ulysses_attention: first all-to-all (peer stores into the symmetric inbox) + the fused "
                "attention reading the inbox; standalone a2a time includes the inbox -> user copy"}
    os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
