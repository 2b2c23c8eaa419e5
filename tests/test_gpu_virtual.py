"""The per-GPU virtual group (Communicator.virtual_group: one rank of a T-rank group at full-GPU
scale, every peer aliasing the rank's own heap, i.e. a self-ring) computes well-defined results,
so the per-GPU measurements run the protocol on correct data paths. On integer data (exact in
bf16 / fp32) at the BASELINE per-rank shapes:
  * AG-GEMM: every step gathers the rank's own slice, so every row block of the output is x @ w;
  * GEMM-RS (ring, fp32 wire): step i adds the GEMM of row slice l_i (ring_indices_rs) to the
    running sum it received from itself, so the output is the sum over all row slices of
    x[slice] @ w (the schedule visits every slice once).
"""
import pytest
import torch

import paper_2604_24013_b200 as tpf

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _ints(shape, lo, hi, seed):
    g = torch.Generator(device=DEV).manual_seed(seed)
    return torch.randint(lo, hi, shape, device=DEV, generator=g, dtype=torch.int32)


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3"])
def test_virtual_tp8_ag_gemm_exact(cfg):
    T = 8
    S, K, N = {"cfg2": (8192, 4096, 28672), "cfg3": (16384, 8192, 10240)}[cfg]
    sl, nl = S // T, N // T
    x = _ints((1, sl, K), 0, 5, 1)
    w = _ints((K, nl), -2, 2, 2)
    want = (x[0].double() @ w.double()).float()
    comm = tpf.Communicator.virtual_group(T, tpf.sym_bytes_ag(T, 1, S, K, nl))
    for _ in range(3):  # both heap parities, and again
        out = torch.full((1, S, nl), float("nan"), device=DEV)
        comm.ag_gemm(x.to(torch.bfloat16), w.to(torch.bfloat16), out)
        comm.sync()
        for r in range(T):
            assert torch.equal(out[0, r * sl:(r + 1) * sl], want), r
    comm.close()


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3"])
def test_virtual_tp8_gemm_rs_ring_exact(cfg):
    T = 8
    S, K, N = {"cfg2": (8192, 14336, 4096), "cfg3": (16384, 8192, 8192)}[cfg]
    kl, sl = K // T, S // T
    x = _ints((1, S, kl), 0, 5, 3)
    w = _ints((kl, N), -2, 2, 4)
    want = (x[0].double() @ w.double()).view(T, sl, N).sum(0).float()  # |sum| < 2^24: exact
    comm = tpf.Communicator.virtual_group(T, tpf.sym_bytes_rs(T, 1, S, kl, N, 1, tpf.F32))
    for _ in range(3):
        out = torch.full((1, sl, N), float("nan"), device=DEV)
        comm.gemm_rs(x.to(torch.bfloat16), w.to(torch.bfloat16), out, kind=tpf.RING, wire=tpf.F32)
        comm.sync()
        assert torch.equal(out[0], want)
    comm.close()


def test_virtual_dp_grad_rs_and_param_ag_exact():
    """cfg 4 per-GPU shapes (8 ranks, 4096 tokens / rank, 2048 x 8192 weight): the gradient RS
    sums the own X^T dY over every row slice of dW; the parameter AG gathers the own weight
    block at every step, so every column block of the output is X . W_own^T."""
    T, M, K, N = 8, 4096, 2048, 8192
    X = _ints((M, K), 0, 5, 5)
    dY = _ints((M, N), -2, 2, 6)
    kl = K // T
    comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_rs(T, 1, K, M, N, 1, tpf.F32),
                                                 tpf.sym_bytes_dp_ag(T, K, N // T)))
    want = (X.double().t() @ dY.double()).view(T, kl, N).sum(0).float()  # < 2^24: exact
    dW = torch.full((kl, N), float("nan"), device=DEV)
    for _ in range(2):
        comm.dp_grad_rs(X.to(torch.bfloat16), dY.to(torch.bfloat16), dW, kind=tpf.RING, wire=tpf.F32)
        comm.sync()
        assert torch.equal(dW, want)
    Nl = N // T
    Wr = _ints((Nl, K), -2, 2, 7)
    blk = (X.double() @ Wr.double().t()).float()
    out = torch.full((M, N), float("nan"), device=DEV)
    for _ in range(2):
        comm.dp_param_ag_gemm(X.to(torch.bfloat16), Wr.to(torch.bfloat16), out)
        comm.sync()
        for j in range(T):
            assert torch.equal(out[:, j * Nl:(j + 1) * Nl], blk), j
    comm.close()


def test_virtual_graph_replay_exact():
    """AG-GEMM and GEMM-RS captured once in a CUDA graph on the virtual group and replayed: the
    device epoch advances per replay, every wait is real, and every replay is exact."""
    T, S, K, N = 8, 2048, 1024, 2048
    sl, nl, kl = S // T, N // T, K // T
    x = _ints((1, sl, K), 0, 5, 8).to(torch.bfloat16)
    w = _ints((K, nl), -2, 2, 9).to(torch.bfloat16)
    xr = _ints((1, S, kl), 0, 5, 10).to(torch.bfloat16)
    wr = _ints((kl, N), -2, 2, 11).to(torch.bfloat16)
    want_ag = (x[0].double() @ w.double()).float()
    want_rs = (xr[0].double() @ wr.double()).view(T, sl, N).sum(0).float()
    y = torch.zeros((1, S, nl), device=DEV)
    yr = torch.zeros((1, sl, N), device=DEV)
    comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, K, nl), tpf.sym_bytes_rs(T, 1, S, kl, N, 1, tpf.F32)))
    s = torch.cuda.Stream(DEV)
    with torch.cuda.stream(s):
        comm.ag_gemm(x, w, y, stream=s)
        comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=tpf.F32, stream=s)
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        comm.ag_gemm(x, w, y, stream=s)
        comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=tpf.F32, stream=s)
    for _ in range(4):
        y.zero_()
        yr.zero_()
        graph.replay()
        torch.cuda.synchronize()
        comm.sync(s)
        for r in range(T):
            assert torch.equal(y[0, r * sl:(r + 1) * sl], want_ag), r
        assert torch.equal(yr[0], want_rs)
    comm.close()
