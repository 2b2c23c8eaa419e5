"""Randomized (fixed-seed) shape / schedule / granularity sweep of the two fused
collectives against the oracle, on integer data (the reference's exact recipe), so every
case must be bit-exact: GPU fp32 accumulation and fp32 wire are exact on these values.
Covers odd group sizes, ragged chunks (rows not a multiple of 128), K / N not multiples
of the tile sizes, B > 1 and m > 1. The DP pair (gradient RS, both wires, through both of its
kernel instances; parameter AG) gets the same treatment. TPF_FUZZ_N=<n> runs n cases per
operator instead of the defaults (a longer sweep)."""
import os

import numpy as np
import pytest
import torch

import paper_2604_24013_b200 as tpf
from test_gpu_parity import DEV, O, bf16, run_ag, run_rs

pytestmark = pytest.mark.gpu
_N = int(os.environ.get("TPF_FUZZ_N", "0"))


def _cases(n, seed, op):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        T = int(rng.integers(1, 9))
        kinds = [tpf.RING, tpf.CIRCULAR] + ([tpf.PAIRWISE] if T % 2 == 0 or T == 1 else [])
        kind = int(rng.choice(kinds))
        m = int(rng.integers(1, 4)) if (op == "ag" or kind == tpf.RING) else 1
        B = int(rng.integers(1, 4))
        S = T * m * int(rng.integers(1, 97))
        if op == "rs":
            K = T * 8 * int(rng.integers(1, 40))
            N = 8 * int(rng.integers(1, 80))
        else:
            K = 8 * int(rng.integers(1, 80))
            N = T * 8 * int(rng.integers(1, 40))
        out.append((T, kind, m, B, S, K, N))
    return out


@pytest.mark.parametrize("T,kind,m,B,S,K,N", _cases(_N or 24, 2026, "rs"))
def test_fuzz_gemm_rs_exact(T, kind, m, B, S, K, N):
    x = O.randint((B, S, K), 0, 5, 11 + S)
    w = O.randint((K, N), -2, 2, 12 + N)
    got = run_rs(T, kind, m, x, w)
    assert np.array_equal(got, O.row_parallel(T, kind, m, x, w))


@pytest.mark.parametrize("T,kind,m,B,S,K,N", _cases(_N or 24, 2027, "ag"))
def test_fuzz_ag_gemm_exact(T, kind, m, B, S, K, N):
    x = O.randint((B, S, K), 0, 5, 13 + S)
    w = O.randint((K, N), -2, 2, 14 + N)
    got = run_ag(T, m, x, w)
    assert np.array_equal(got, O.column_parallel(T, m, x, w))


def _dp_cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        T = int(rng.integers(1, 9))
        kinds = [tpf.RING, tpf.CIRCULAR] + ([tpf.PAIRWISE] if T % 2 == 0 or T == 1 else [])
        kind = int(rng.choice(kinds))
        m = int(rng.integers(1, 3)) if kind == tpf.RING else 1
        M = 8 * int(rng.integers(1, 33))           # tokens per rank (the GEMM's K)
        K = T * m * 8 * int(rng.integers(1, 40))   # dW rows, scattered over the ranks
        N = 8 * int(rng.integers(1, 80))
        wire = int(rng.choice([tpf.F32, tpf.BF16]))
        out.append((T, kind, m, M, K, N, wire))
    return out


@pytest.mark.parametrize("T,kind,m,M,K,N,wire", _dp_cases(_N or 16, 2028))
def test_fuzz_dp_grad_rs_exact(T, kind, m, M, K, N, wire):
    """dW = sum_q X_q^T dY_q reduce-scattered by rows, every schedule and both wires (the
    pairwise bf16 case runs the staged-fold instance): exact against the oracle. For the bf16
    wire the data keeps every partial within bf16's exact integers."""
    hi = (2, 2) if wire == tpf.BF16 else (5, 2)
    X = np.stack([O.randint((M, K), 0, hi[0], 300 + r + M) for r in range(T)])
    dY = np.stack([O.randint((M, N), 1 - hi[1], hi[1], 400 + r + N) for r in range(T)])
    parts = np.stack([(X[r].T @ dY[r])[None] for r in range(T)])
    if wire == tpf.BF16:
        assert np.abs(parts).max() <= 256
    Xd = torch.stack([bf16(X[r]) for r in range(T)]).to(DEV)
    dYd = torch.stack([bf16(dY[r]) for r in range(T)]).to(DEV)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_rs(T, 1, K, M, N, m, wire))
    dW = torch.full((T, K // T, N), float("nan"), device=DEV)
    comm.dp_grad_rs(Xd, dYd, dW, kind=kind, m=m, wire=wire)
    comm.sync()
    comm.close()
    assert np.array_equal(dW.double().cpu().numpy(), O.fuse_rs_identity(T, kind, m, parts)[:, 0])


@pytest.mark.parametrize("T,M,K,Nl", [(int(t), int(a), int(b), int(c)) for t, a, b, c in zip(
    *(np.random.default_rng(2029).integers(lo, hi, _N or 12) for lo, hi in ((1, 9), (1, 300), (1, 60), (1, 40))))])
def test_fuzz_dp_param_ag_gemm_exact(T, M, K, Nl):
    """DP parameter AG fused into the forward GEMM on ragged shapes: out_r = x_r . W^T."""
    K, Nl = 8 * K, 8 * Nl
    X = np.stack([O.randint((M, K), 0, 3, 500 + r + M) for r in range(T)])
    W = O.randint((Nl * T, K), -2, 2, 600 + K)
    xd = torch.stack([bf16(X[r]) for r in range(T)]).to(DEV)
    wd = torch.stack([bf16(W[r * Nl:(r + 1) * Nl]) for r in range(T)]).to(DEV)
    out = torch.full((T, M, Nl * T), float("nan"), device=DEV)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_dp_ag(T, K, Nl))
    comm.dp_param_ag_gemm(xd, wd, out)
    comm.sync()
    comm.close()
    assert np.array_equal(out.double().cpu().numpy(), np.stack([X[r] @ W.T for r in range(T)]))
