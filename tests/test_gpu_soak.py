"""Soak test: one communicator, a seeded random sequence of every fused operator (both heap
parities, every schedule, graph replays in between), each result checked. Catches any
cross-operator interference through the shared flag / heap regions and the device epoch."""
import os

import numpy as np
import pytest
import torch

import paper_2604_24013_b200 as tpf
from test_gpu_parity import DEV, O, bf16

pytestmark = pytest.mark.gpu


def test_mixed_operator_sequence_on_one_communicator():
    # TPF_SOAK="T,steps" for a longer run (default 4 ranks, 40 steps)
    T, steps = (int(v) for v in os.environ.get("TPF_SOAK", "4,40").split(","))
    B, S, D, H = 1, 128 * T, 256, 128 * T
    heads, Dh = 4, 128
    rng = np.random.default_rng(2027)
    Md = 96  # DP tokens per rank
    need = max(tpf.sym_bytes_ag(T, B, S, D, H // T), tpf.sym_bytes_rs(T, B, S, H // T, D, 2),
               tpf.sym_bytes_ulysses(T, B, heads * T, S, Dh), tpf.sym_bytes_dp_ag(T, D, H // T),
               tpf.sym_bytes_rs(T, 1, D, Md, H, 1, tpf.BF16))
    comm = tpf.Communicator.local_group(T, need)
    ref = tpf.Communicator.local_group(T, need)  # a second group computes eager references
    s = torch.cuda.Stream(DEV)

    # operands
    xa = O.randint((B, S, D), 0, 3, 1)
    wa = O.randint((D, H), -2, 2, 2)
    xa_d = torch.stack([bf16(xa[:, r * (S // T):(r + 1) * (S // T)]) for r in range(T)]).to(DEV)
    wa_d = torch.stack([bf16(wa[:, r * (H // T):(r + 1) * (H // T)]) for r in range(T)]).to(DEV)
    xr = O.randint((B, S, H), 0, 3, 3)
    wr = O.randint((H, D), -2, 2, 4)
    xr_d = torch.stack([bf16(xr[:, :, r * (H // T):(r + 1) * (H // T)]) for r in range(T)]).to(DEV)
    wr_d = torch.stack([bf16(wr[r * (H // T):(r + 1) * (H // T)]) for r in range(T)]).to(DEV)
    g = torch.Generator(device=DEV).manual_seed(6)
    hq = [torch.randn((T, B * heads, S, Dh), device=DEV, generator=g).to(torch.bfloat16) for _ in range(3)]
    sq = [torch.randn((T, B * heads * T, S // T, Dh), device=DEV, generator=g).to(torch.bfloat16) for _ in range(3)]

    want_ag = O.column_parallel(T, 1, xa, wa)
    out_ag = torch.empty((T, B, S, H // T), device=DEV)

    def run_ag(c):
        c.ag_gemm(xa_d, wa_d, out_ag, stream=s)
        return lambda: np.array_equal(out_ag.double().cpu().numpy(), want_ag)

    wants_rs = {(k, m): O.row_parallel(T, k, m, xr, wr) for k in (tpf.RING, tpf.PAIRWISE, tpf.CIRCULAR)
                for m in ((1, 2) if k == tpf.RING else (1,))}
    out_rs = torch.empty((T, B, S // T, D), device=DEV)

    def run_rs(c, k, m):
        c.gemm_rs(xr_d, wr_d, out_rs, kind=k, m=m, stream=s)
        return lambda: np.array_equal(out_rs.double().cpu().numpy(), wants_rs[(k, m)])

    def eager(fn_ref, out):
        with torch.cuda.stream(s):
            fn_ref(ref)
        torch.cuda.synchronize()
        return out.clone()

    out_a2a = torch.empty((T, B, S // T, T * heads * Dh), device=DEV, dtype=torch.bfloat16)
    want_a2a = eager(lambda c: c.attention_a2a(*hq, out_a2a, B, heads, stream=s), out_a2a)
    out_ul = torch.empty((T, B, S // T, heads * T * Dh), device=DEV, dtype=torch.bfloat16)
    want_ul = eager(lambda c: c.ulysses_attention(*sq, out_ul, B, heads * T, stream=s), out_ul)

    def run_a2a(c):
        c.attention_a2a(*hq, out_a2a, B, heads, stream=s)
        return lambda: torch.equal(out_a2a, want_a2a)

    def run_ul(c):
        c.ulysses_attention(*sq, out_ul, B, heads * T, stream=s)
        return lambda: torch.equal(out_ul, want_ul)

    # DP ops (cfg 4 family): the gradient RS through both of its kernel instances (ring, and the
    # pairwise one over the bf16 wire: small-integer partials bf16 holds exactly) and the
    # parameter AG fused into the forward GEMM
    Xg = O.randint((T, Md, D), 0, 2, 7)
    dYg = O.randint((T, Md, H), -1, 2, 8)
    parts = np.stack([(Xg[r].T @ dYg[r])[None] for r in range(T)])
    dp_kinds = [tpf.RING] + ([tpf.PAIRWISE] if T % 2 == 0 else [])
    wants_dp = {k: O.fuse_rs_identity(T, k, 1, parts)[:, 0] for k in dp_kinds}
    Xg_d = torch.stack([bf16(Xg[r]) for r in range(T)]).to(DEV)
    dYg_d = torch.stack([bf16(dYg[r]) for r in range(T)]).to(DEV)
    out_dp = torch.empty((T, D // T, H), device=DEV)

    def run_dp(c, k):
        c.dp_grad_rs(Xg_d, dYg_d, out_dp, kind=k, wire=tpf.BF16, stream=s)
        return lambda: np.array_equal(out_dp.double().cpu().numpy(), wants_dp[k])

    Wp = O.randint((H, D), -2, 2, 9)  # (N = Nl * T, K), row-sharded (PyTorch Linear layout)
    Wp_d = torch.stack([bf16(Wp[r * (H // T):(r + 1) * (H // T)]) for r in range(T)]).to(DEV)
    want_pa = np.stack([Xg[r] @ Wp.T for r in range(T)])
    out_pa = torch.empty((T, Md, H), device=DEV)

    def run_pa(c):
        c.dp_param_ag_gemm(Xg_d, Wp_d, out_pa, stream=s)
        return lambda: np.array_equal(out_pa.double().cpu().numpy(), want_pa)

    ops = [lambda c: run_ag(c), lambda c: run_a2a(c), lambda c: run_ul(c), lambda c: run_pa(c)]
    ops += [(lambda k, m: (lambda c: run_rs(c, k, m)))(k, m) for (k, m) in wants_rs]
    ops += [(lambda k: (lambda c: run_dp(c, k)))(k) for k in dp_kinds]

    # a captured graph of two different collectives, replayed in the middle of the sequence
    with torch.cuda.stream(s):
        run_ag(comm)
        run_rs(comm, tpf.RING, 1)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        run_ag(comm)
        run_rs(comm, tpf.RING, 1)

    for step in range(steps):
        if step % 7 == 3:
            out_ag.zero_()
            out_rs.zero_()
            graph.replay()
            torch.cuda.synchronize()
            assert np.array_equal(out_ag.double().cpu().numpy(), want_ag), step
            assert np.array_equal(out_rs.double().cpu().numpy(), wants_rs[(tpf.RING, 1)]), step
            continue
        op = ops[int(rng.integers(len(ops)))]
        with torch.cuda.stream(s):
            check = op(comm)
        torch.cuda.synchronize()
        assert check(), step
    comm.sync()
    comm.close()
    ref.close()
