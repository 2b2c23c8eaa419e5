"""The one-process-per-GPU code path with real peer waits, on one GPU (split group).

`Communicator.split_group(T)` builds T per-rank communicators exactly as T processes would
(tpf_comm_create: own symmetric heap, own device epoch, own error record), with the peers'
heaps mapped directly instead of through CUDA IPC. Every fused GEMM call is made per rank with
that rank's own tensors; the launch parameters are the per-process ones (one hosted rank,
rank id r, per-rank tensor maps over the rank's own heap), and the last rank's call runs all
ranks as ONE launch (ranks whose kernels wait on each other must not be separate launches on
one GPU). So these tests run the per-rank protocol -- peer stores into other heaps, per-rank
flags and epochs, flag waits, blame tables -- that the multi-GPU path runs, and check it
bit-exactly against the oracle / the reference's own golden outputs (integer data).

References: fabric.cpp:9-103 (send/recv/wait), fabric.hpp:185-226 (spawn_group, GroupError),
acceptance_test.cpp:99-187 (C1), collectives_test.cpp:249-294.
"""
import numpy as np
import pytest
import torch

import paper_2604_24013_b200 as tpf
from test_gpu_fuzz import _cases
from test_gpu_parity import _TAGS, _Z, DEV, O, bf16, run_ag, run_rs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag", _TAGS)
def test_split_c1_row_parallel_exact_vs_reference_golden(tag):
    t, kind, m = (int(tag.split("_")[i][1:]) for i in range(3))
    got = run_rs(t, kind, m, _Z[f"{tag}/x2"], _Z[f"{tag}/w2"], split=True)
    assert np.array_equal(got, _Z[f"{tag}/row"]), np.abs(got - _Z[f"{tag}/row"]).max()


@pytest.mark.parametrize("tag", _TAGS)
def test_split_c1_column_parallel_exact_vs_reference_golden(tag):
    t, kind, m = (int(tag.split("_")[i][1:]) for i in range(3))
    got = run_ag(t, m, _Z[f"{tag}/x"], _Z[f"{tag}/up"], split=True)
    assert np.array_equal(got, _Z[f"{tag}/col"])


@pytest.mark.parametrize("T,kind,m,B,S,K,N", _cases(24, 2026, "rs"))
def test_split_fuzz_gemm_rs_exact(T, kind, m, B, S, K, N):
    x = O.randint((B, S, K), 0, 5, 11 + S)
    w = O.randint((K, N), -2, 2, 12 + N)
    assert np.array_equal(run_rs(T, kind, m, x, w, split=True), O.row_parallel(T, kind, m, x, w))


@pytest.mark.parametrize("T,kind,m,B,S,K,N", _cases(24, 2027, "ag"))
def test_split_fuzz_ag_gemm_exact(T, kind, m, B, S, K, N):
    x = O.randint((B, S, K), 0, 5, 13 + S)
    w = O.randint((K, N), -2, 2, 14 + N)
    assert np.array_equal(run_ag(T, m, x, w, split=True), O.column_parallel(T, m, x, w))


@pytest.mark.parametrize("T", [2, 4, 8])
def test_split_repeated_calls_reverse_rank_order(T):
    """Per-rank epochs advance call by call (both heap parities reused) and the ranks may
    make their calls in any order: rank T-1 first here, as threads of spawn_group would."""
    B, S, K, N = 1, 128 * T, 64 * T, 256
    x = O.randint((B, S, K), 0, 5, 21)
    w = O.randint((K, N), -2, 2, 22)
    kl = K // T
    xs = torch.stack([bf16(x[:, :, r * kl:(r + 1) * kl]) for r in range(T)]).to(DEV)
    ws = torch.stack([bf16(w[r * kl:(r + 1) * kl]) for r in range(T)]).to(DEV)
    comms = tpf.Communicator.split_group(T, tpf.sym_bytes_rs(T, B, S, kl, N))
    for kind in (tpf.RING, tpf.CIRCULAR, tpf.PAIRWISE, tpf.RING, tpf.PAIRWISE):
        out = torch.full((T, B, S // T, N), float("nan"), device=DEV)
        for r in reversed(range(T)):
            comms[r].gemm_rs(xs[r], ws[r], out[r], kind=kind)
        for c in comms:
            c.sync()
        assert np.array_equal(out.double().cpu().numpy(), O.row_parallel(T, kind, 1, x, w)), kind
    for c in comms:
        c.close()


@pytest.mark.parametrize("T", [2, 4, 8])
def test_split_dp_grad_rs_and_param_ag_exact(T):
    """DP gradient RS and parameter AG (cfg 4, a19) through the per-rank path."""
    M, K, N = 96, 64 * T, 136
    X = np.stack([O.randint((M, K), 0, 5, 60 + r) for r in range(T)])
    dY = np.stack([O.randint((M, N), -2, 2, 70 + r) for r in range(T)])
    parts = np.stack([(X[r].T @ dY[r])[None] for r in range(T)])
    Xd = torch.stack([bf16(X[r]) for r in range(T)]).to(DEV)
    dYd = torch.stack([bf16(dY[r]) for r in range(T)]).to(DEV)
    comms = tpf.Communicator.split_group(T, max(tpf.sym_bytes_rs(T, 1, K, M, N, 1), tpf.sym_bytes_dp_ag(T, K, 64)))
    for kind in (tpf.RING, tpf.PAIRWISE, tpf.CIRCULAR):
        dW = torch.full((T, K // T, N), float("nan"), device=DEV)
        for r in range(T):
            comms[r].dp_grad_rs(Xd[r], dYd[r], dW[r], kind=kind)
        for c in comms:
            c.sync()
        assert np.array_equal(dW.double().cpu().numpy(), O.fuse_rs_identity(T, kind, 1, parts)[:, 0]), kind
    Nl = 64
    W = O.randint((Nl * T, K), -2, 2, 90)
    wd = torch.stack([bf16(W[r * Nl:(r + 1) * Nl]) for r in range(T)]).to(DEV)
    out = torch.full((T, M, Nl * T), float("nan"), device=DEV)
    for r in range(T):
        comms[r].dp_param_ag_gemm(Xd[r], wd[r], out[r])
    for c in comms:
        c.sync()
    got = out.double().cpu().numpy()
    for r in range(T):
        assert np.array_equal(got[r], X[r] @ W.T), r
    for c in comms:
        c.close()


@pytest.mark.parametrize("op", ["rs_ring", "rs_pairwise", "rs_circular", "ag"])
@pytest.mark.parametrize("bad", [1, 3])
def test_split_failed_rank_names_the_failing_rank(op, bad):
    """Fault injection on the per-rank path: every rank that reports an error reports
    GroupError naming the rank that stopped publishing (fabric_test.cpp:44-58), each from its
    own error record and its own copy of the blame table; the group recovers afterwards."""
    T, B, S, K, N = 4, 1, 512, 256, 256
    comms = tpf.Communicator.split_group(T, tpf.sym_bytes_rs(T, B, S, K, N, 1) + tpf.sym_bytes_ag(T, B, S, K, N, 1))
    for c in comms:
        c.set_timeout_ms(200)
        c.inject_fault(bad)
    x = O.randint((B, S, K), 0, 5, 1)
    w = O.randint((K, N), -2, 2, 2)
    kind = {"rs_ring": tpf.RING, "rs_pairwise": tpf.PAIRWISE, "rs_circular": tpf.CIRCULAR}.get(op)
    sl, nl, kl = S // T, N // T, K // T
    xa = torch.stack([bf16(x[:, r * sl:(r + 1) * sl]) for r in range(T)]).to(DEV)
    wa = torch.stack([bf16(w[:, r * nl:(r + 1) * nl]) for r in range(T)]).to(DEV)
    oa = torch.empty((T, B, S, nl), device=DEV)
    xr = torch.stack([bf16(x[:, :, r * kl:(r + 1) * kl]) for r in range(T)]).to(DEV)
    wr = torch.stack([bf16(w[r * kl:(r + 1) * kl]) for r in range(T)]).to(DEV)
    orr = torch.empty((T, B, S // T, N), device=DEV)

    def call():
        for r in range(T):
            if op == "ag":
                comms[r].ag_gemm(xa[r], wa[r], oa[r])
            else:
                comms[r].gemm_rs(xr[r], wr[r], orr[r], kind=kind)

    call()
    reported = []
    for c in comms:
        try:
            c.sync()
        except tpf.GroupError as e:
            reported.append(e.failing_rank())
    assert reported and all(f == bad for f in reported), reported
    for c in comms:
        c.inject_fault(-1)
    call()
    for c in comms:
        c.sync()
    if op == "ag":
        assert np.array_equal(oa.double().cpu().numpy(), O.column_parallel(T, 1, x, w))
    else:
        assert np.array_equal(orr.double().cpu().numpy(), O.row_parallel(T, kind, 1, x, w))
    for c in comms:
        c.close()


def test_split_group_rejects_mismatched_and_incomplete_calls():
    """Calls are collective: a rank calling twice before the others, or a different call,
    is refused (and the group resets); sync with a call still pending is refused."""
    T, B, S, K, N = 2, 1, 256, 128, 256
    comms = tpf.Communicator.split_group(T, tpf.sym_bytes_rs(T, B, S, K, N, 1) + tpf.sym_bytes_ag(T, B, S, K, N, 1))
    x = torch.zeros((B, S, K // T), device=DEV, dtype=torch.bfloat16)
    w = torch.zeros((K // T, N), device=DEV, dtype=torch.bfloat16)
    out = torch.zeros((B, S // T, N), device=DEV)
    comms[0].gemm_rs(x, w, out)
    with pytest.raises(ValueError, match="still waiting"):
        comms[0].sync()
    with pytest.raises(ValueError, match="second call"):
        comms[0].gemm_rs(x, w, out)
    comms[0].gemm_rs(x, w, out, kind=tpf.RING)
    with pytest.raises(ValueError, match="different collective call"):
        comms[1].gemm_rs(x, w, out, kind=tpf.PAIRWISE)
    for r in range(T):
        comms[r].gemm_rs(x, w, out)
    for c in comms:
        c.sync()
    with pytest.raises(ValueError, match="split group"):
        q = torch.zeros((2, S, 128), device=DEV, dtype=torch.bfloat16)
        comms[0].attention_a2a(q, q, q, torch.zeros((1, S // T, T * 2 * 128), device=DEV, dtype=torch.bfloat16), 1, 2)
    for c in comms:
        c.close()


def test_split_group_cuda_graph_replay():
    """The deferred launch is issued by the last rank's call, so a graph captured around the
    T per-rank calls holds the one group launch and replays with device-side epochs."""
    T, B, S, K, N = 4, 1, 512, 256, 256
    x = O.randint((B, S, K), 0, 5, 31)
    w = O.randint((K, N), -2, 2, 32)
    kl = K // T
    xs = torch.stack([bf16(x[:, :, r * kl:(r + 1) * kl]) for r in range(T)]).to(DEV)
    ws = torch.stack([bf16(w[r * kl:(r + 1) * kl]) for r in range(T)]).to(DEV)
    out = torch.zeros((T, B, S // T, N), device=DEV)
    comms = tpf.Communicator.split_group(T, tpf.sym_bytes_rs(T, B, S, kl, N))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for r in range(T):  # eager warm-up call (epoch 1)
            comms[r].gemm_rs(xs[r], ws[r], out[r], stream=s)
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for r in range(T):
            comms[r].gemm_rs(xs[r], ws[r], out[r], stream=s)
    want = O.row_parallel(T, tpf.RING, 1, x, w)
    for _ in range(3):
        out.zero_()
        graph.replay()
        torch.cuda.synchronize()
        for c in comms:
            c.sync(s)
        assert np.array_equal(out.double().cpu().numpy(), want)
    for c in comms:
        c.close()
