"""Full-size parity at every BASELINE configuration (cfg1, cfg2, cfg3), bit-exact.

The reference's exactness contract (acceptance_test.cpp:99-187, C1; collectives_test.cpp:270-294,
cross-schedule byte identity) is checked here at the BASELINE shapes themselves, not only at the
small golden sizes:

* data: the reference's integer recipe (x in [0,5), w in [-2,2); experiment.cpp:163-168), drawn
  on the device. Every product and every partial sum is an integer of magnitude
  <= 8 * K < 2^24, so bf16 operands, fp32 accumulation, the fp32 wire and fp32 outputs are all
  exact and the result is independent of summation order -- any correct schedule must equal the
  exact product bit for bit;
* checker: the exact product in fp64 on the device (cuBLAS DGEMM; integers < 2^53 are exact in
  any order, so it equals the fp64 oracle's result), plus a few full rows through the C oracle
  itself (oracle/tpf_oracle.c, matmul = tensor.cpp:68-85) to tie the two checkers together;
* group: the single-GPU local group (all T ranks in one launch), and for cfg1 / cfg3 at T = 8
  the split group too (the per-rank, one-process-per-GPU code path).
"""
import numpy as np
import pytest
import torch

import paper_2604_24013_b200 as tpf
from test_gpu_parity import DEV, O

pytestmark = pytest.mark.gpu

# (name, T, S, K, N): AG-GEMM gathers S (K features) and computes N/T columns per rank;
# GEMM-RS reduces K/T per rank and scatters S.
AG_CASES = [
    ("cfg1", 4, 4096, 4096, 4096),
    ("cfg2_gate_up", 8, 8192, 4096, 28672),
    ("cfg3_qkv_T2", 2, 16384, 8192, 10240),
    ("cfg3_qkv_T4", 4, 16384, 8192, 10240),
    ("cfg3_qkv_T8", 8, 16384, 8192, 10240),
]
RS_CASES = [
    ("cfg1", 4, 4096, 4096, 4096),
    ("cfg2_down", 8, 8192, 14336, 4096),
    ("cfg3_out_T2", 2, 16384, 8192, 8192),
    ("cfg3_out_T4", 4, 16384, 8192, 8192),
    ("cfg3_out_T8", 8, 16384, 8192, 8192),
]


def _ints(shape, lo, hi, seed):
    g = torch.Generator(device=DEV).manual_seed(seed)
    return torch.randint(lo, hi, shape, device=DEV, generator=g, dtype=torch.int32)


def _oracle_rows(x_rows, w):
    """A few rows through the C oracle's matmul (fp64, the reference's loop order)."""
    return O.matmul(x_rows.double().cpu().numpy(), w.double().cpu().numpy())


def _kinds(T):
    return [tpf.RING, tpf.CIRCULAR] + ([tpf.PAIRWISE] if T % 2 == 0 else [])


@pytest.mark.parametrize("name,T,S,K,N", AG_CASES, ids=[c[0] for c in AG_CASES])
def test_fullsize_ag_gemm_exact(name, T, S, K, N):
    x = _ints((S, K), 0, 5, 1)
    w = _ints((K, N), -2, 2, 2)
    want = x.double() @ w.double()  # exact integers
    sl, nl = S // T, N // T
    xs = x.reshape(T, 1, sl, K).to(torch.bfloat16)
    ws = w.reshape(K, T, nl).permute(1, 0, 2).contiguous().to(torch.bfloat16)
    out = torch.full((T, 1, S, nl), float("nan"), device=DEV)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ag(T, 1, S, K, nl, 1))
    comm.ag_gemm(xs, ws, out)
    comm.sync()
    comm.close()
    for r in range(T):
        assert torch.equal(out[r, 0].double(), want[:, r * nl:(r + 1) * nl]), (name, r)
    rows = torch.tensor([0, S // 2 + 17, S - 1], device=DEV)
    assert np.array_equal(out[T - 1, 0, rows].double().cpu().numpy(),
                          _oracle_rows(x[rows], w[:, (T - 1) * nl:]))
    del out, xs, ws, want
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,T,S,K,N", RS_CASES, ids=[c[0] for c in RS_CASES])
def test_fullsize_gemm_rs_exact_every_schedule(name, T, S, K, N):
    """Every schedule at full size, fp32 wire: bit-exact and byte-identical across schedules
    (collectives_test.cpp:270-294 at the BASELINE shapes)."""
    x = _ints((S, K), 0, 5, 3)
    w = _ints((K, N), -2, 2, 4)
    want = x.double() @ w.double()
    kl, sl = K // T, S // T
    xs = x.reshape(S, T, kl).permute(1, 0, 2).reshape(T, 1, S, kl).contiguous().to(torch.bfloat16)
    ws = w.reshape(T, kl, N).to(torch.bfloat16)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_rs(T, 1, S, kl, N, 1, tpf.F32))
    outs = []
    for kind in _kinds(T):
        out = torch.full((T, 1, sl, N), float("nan"), device=DEV)
        comm.gemm_rs(xs, ws, out, kind=kind, wire=tpf.F32)
        comm.sync()
        for r in range(T):
            assert torch.equal(out[r, 0].double(), want[r * sl:(r + 1) * sl]), (name, kind, r)
        outs.append(out)
    comm.close()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    rows = torch.tensor([0, sl - 1], device=DEV)
    assert np.array_equal(outs[0][1, 0, rows].double().cpu().numpy(), _oracle_rows(x[sl + rows], w))
    del outs, xs, ws, want
    torch.cuda.empty_cache()


def test_fullsize_cfg1_ring_granularity2_exact():
    """cfg1 with m = 2 (the ring's chunk granularity, collectives.cpp:374-398) for both ops."""
    T, S, K, N = 4, 4096, 4096, 4096
    x = _ints((S, K), 0, 5, 5)
    w = _ints((K, N), -2, 2, 6)
    want = x.double() @ w.double()
    kl, sl, nl = K // T, S // T, N // T
    xs = x.reshape(S, T, kl).permute(1, 0, 2).reshape(T, 1, S, kl).contiguous().to(torch.bfloat16)
    ws = w.reshape(T, kl, N).to(torch.bfloat16)
    comm = tpf.Communicator.local_group(T, max(tpf.sym_bytes_rs(T, 1, S, kl, N, 2, tpf.F32),
                                               tpf.sym_bytes_ag(T, 1, S, K, nl, 2)))
    out = torch.full((T, 1, sl, N), float("nan"), device=DEV)
    comm.gemm_rs(xs, ws, out, kind=tpf.RING, m=2, wire=tpf.F32)
    comm.sync()
    for r in range(T):
        assert torch.equal(out[r, 0].double(), want[r * sl:(r + 1) * sl]), r
    xa = x.reshape(T, 1, sl, K).to(torch.bfloat16)
    wa = w.reshape(K, T, nl).permute(1, 0, 2).contiguous().to(torch.bfloat16)
    oa = torch.full((T, 1, S, nl), float("nan"), device=DEV)
    comm.ag_gemm(xa, wa, oa, m=2)
    comm.sync()
    comm.close()
    for r in range(T):
        assert torch.equal(oa[r, 0].double(), want[:, r * nl:(r + 1) * nl]), r


@pytest.mark.parametrize("name,T,S,K,N", [AG_CASES[0], AG_CASES[4]], ids=["cfg1", "cfg3_qkv_T8"])
def test_fullsize_split_group_ag_exact(name, T, S, K, N):
    """The per-rank (one process per GPU) launch path at full size: each rank's own call, own
    heap, epoch and flags, all ranks in one grid (tpf_comm_create_split_group)."""
    x = _ints((S, K), 0, 5, 7)
    w = _ints((K, N), -2, 2, 8)
    want = x.double() @ w.double()
    sl, nl = S // T, N // T
    xs = x.reshape(T, 1, sl, K).to(torch.bfloat16)
    ws = w.reshape(K, T, nl).permute(1, 0, 2).contiguous().to(torch.bfloat16)
    out = torch.full((T, 1, S, nl), float("nan"), device=DEV)
    comms = tpf.Communicator.split_group(T, tpf.sym_bytes_ag(T, 1, S, K, nl, 1))
    for r in range(T):
        comms[r].ag_gemm(xs[r], ws[r], out[r])
    for c in comms:
        c.sync()
        c.close()
    for r in range(T):
        assert torch.equal(out[r, 0].double(), want[:, r * nl:(r + 1) * nl]), (name, r)


@pytest.mark.parametrize("name,T,S,K,N", [RS_CASES[0], RS_CASES[4]], ids=["cfg1", "cfg3_out_T8"])
def test_fullsize_split_group_gemm_rs_exact(name, T, S, K, N):
    x = _ints((S, K), 0, 5, 9)
    w = _ints((K, N), -2, 2, 10)
    want = x.double() @ w.double()
    kl, sl = K // T, S // T
    xs = x.reshape(S, T, kl).permute(1, 0, 2).reshape(T, 1, S, kl).contiguous().to(torch.bfloat16)
    ws = w.reshape(T, kl, N).to(torch.bfloat16)
    comms = tpf.Communicator.split_group(T, tpf.sym_bytes_rs(T, 1, S, kl, N, 1, tpf.F32))
    for kind in (tpf.RING, tpf.PAIRWISE):
        out = torch.full((T, 1, sl, N), float("nan"), device=DEV)
        for r in range(T):
            comms[r].gemm_rs(xs[r], ws[r], out[r], kind=kind, wire=tpf.F32)
        for c in comms:
            c.sync()
        for r in range(T):
            assert torch.equal(out[r, 0].double(), want[r * sl:(r + 1) * sl]), (name, kind, r)
    for c in comms:
        c.close()


@pytest.mark.parametrize("kind", [tpf.RING, tpf.PAIRWISE, tpf.CIRCULAR])
def test_query_split_attention_T8_vs_oracle(kind):
    """Query-split attention (Alg. 4) at T = 8, the group size cfg3 runs it at, every schedule;
    rel_deviation <= 2e-2 (bf16 P and context) vs the fp64 oracle."""
    from test_gpu_parity import bf16, bf16_round, rel_deviation
    T, batch, heads, Dh, D = 8, 1, 1, 128, 256
    S = 128 * T
    rng = np.random.default_rng(900 + kind)
    q, k, v = (bf16_round(rng.uniform(-1, 1, (T, batch * heads, S, Dh))) for _ in range(3))
    w_o = bf16_round(rng.uniform(-1, 1, (T * heads * Dh, D)) / 16)
    dq, dk, dv = (bf16(a).to(DEV) for a in (q, k, v))
    dw = bf16(w_o.reshape(T, heads * Dh, D)).to(DEV)
    out = torch.empty((T, batch, S // T, D), device=DEV)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_rs(T, batch, S, heads * Dh, D, 1) + (1 << 22))
    comm.query_split_attention(dq, dk, dv, dw, out, batch, heads, kind=kind)
    comm.sync()
    comm.close()
    want = O.query_split_attention(T, kind, batch, heads, q, k, v, w_o)
    assert rel_deviation(out.double().cpu().numpy(), want) <= 2e-2


@pytest.mark.parametrize("M,K,N", [(8192, 4096, 28672), (8192, 14336, 4096), (4096, 4096, 4864), (2048, 8192, 1280)],
                         ids=["bench_up_wide", "bench_down_narrow", "narrow_partial_group", "cfg3_qkv_per_rank"])
def test_fullsize_t1_gemm_exact(M, K, N):
    """The T = 1 GEMM (MODE_SINGLE) at the bench block's shapes and through the raster paths its
    heuristics pick (tpf_runtime.cu: wide N -> evict_last A panels; narrow N -> group_n n-tile
    sweeps with an evict_last B slab, including a last group of fewer n-tiles): exact integer
    product in fp32 (|sums| < 2^24)."""
    x = _ints((M, K), 0, 5, 11)
    w = _ints((K, N), -2, 2, 12)
    out = torch.full((M, N), float("nan"), device=DEV)
    tpf.gemm(x.to(torch.bfloat16), w.to(torch.bfloat16), out)
    torch.cuda.synchronize()
    assert torch.equal(out.double(), x.double() @ w.double())


def test_fullsize_t1_swiglu_bench_shape():
    """The bench block's first GEMM as the bench runs it: T = 1, 8192 x 4096 x (2 x 14336) with
    SwiGLU fused in the epilogue over the tile-interleaved gate||up weight, bf16 output, against
    an fp32 torch reference (bf16 output rounding: 1e-2 of the max)."""
    S, D, F = 8192, 4096, 14336
    g = torch.Generator(device=DEV).manual_seed(21)
    x = torch.randn((1, S, D), device=DEV, generator=g).to(torch.bfloat16)
    gate = (torch.randn((D, F), device=DEV, generator=g) / D ** 0.5).to(torch.bfloat16)
    up = (torch.randn((D, F), device=DEV, generator=g) / D ** 0.5).to(torch.bfloat16)
    w = tpf.interleave_gate_up(gate, up).contiguous()
    out = torch.empty((1, S, F), device=DEV, dtype=torch.bfloat16)
    one = tpf.Communicator.create(0, 1, 0)
    one.ag_gemm(x, w, out, act=tpf.ACT_SWIGLU)
    one.sync()
    one.close()
    xf = x[0].float()
    for c0 in (0, F // 2, F - 2048):  # three column bands keep the fp32 reference small
        ref = torch.nn.functional.silu(xf @ gate[:, c0:c0 + 2048].float()) * (xf @ up[:, c0:c0 + 2048].float())
        err = (out[0, :, c0:c0 + 2048].float() - ref).abs().max().item()
        assert err <= 1e-2 * ref.abs().max().item(), (c0, err)
