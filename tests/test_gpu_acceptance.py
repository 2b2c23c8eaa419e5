"""GPU analogues of the reference's acceptance criteria C4 (no tail) and C6 (overlap).

C4 (acceptance_test.cpp:291-307, costmodel.cpp:163-176 no_tail_check): on the reference's
simulated timeline no communication interval of a rank ends after its last compute interval.
Here the same predicate is evaluated on the kernel's own %globaltimer records
(paper_2604_24013_b200.trace): per rank, the last peer-flag publication (GEMM-RS partial
pushed to the successor, AG image forwarded) against the end of that rank's last GEMM tile.
It is asserted for every op x schedule x group size, in the single-GPU local group (all ranks
in one launch), in the split group (the per-rank launch path) and in the per-GPU virtual
group (one rank of a TP group at full scale).

C6 (acceptance_test.cpp:334-366: fused <= 1.25 x pure compute): the per-GPU fused op of a
TP = 8 group (virtual peers, full cfg2 / cfg3 per-rank shapes) against the plain T = 1 GEMM of
the same per-rank shapes. NVLink is not in this measurement (one GPU); the protocol's on-GPU
cost -- wire images, forwarding, inbox reads, flags and waits -- is.
"""
import pytest
import torch

import paper_2604_24013_b200 as tpf
from paper_2604_24013_b200 import trace

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _traced(comm, call):
    for _ in range(2):
        call()
    comm.sync()
    buf = trace.alloc(300000)
    comm.set_trace(buf)
    call()
    comm.sync()
    comm.set_trace(None)
    recs = trace.decode(buf)
    assert 0 < len(recs) < 300000
    return trace.summarize(recs)


def _kinds(T):
    return [tpf.RING, tpf.CIRCULAR] + ([tpf.PAIRWISE] if T % 2 == 0 else [])


def _tensors(T, S, K, N, lead):
    g = torch.Generator(device=DEV).manual_seed(T)
    L = (T,) if lead else ()
    xa = torch.randn(L + (1, S // T, K), device=DEV, generator=g).to(torch.bfloat16)
    wa = (torch.randn(L + (K, N // T), device=DEV, generator=g) / 32).to(torch.bfloat16)
    oa = torch.empty(L + (1, S, N // T), device=DEV, dtype=torch.bfloat16)
    xr = torch.randn(L + (1, S, K // T), device=DEV, generator=g).to(torch.bfloat16)
    wr = (torch.randn(L + (K // T, N), device=DEV, generator=g) / 32).to(torch.bfloat16)
    orr = torch.empty(L + (1, S // T, N), device=DEV, dtype=torch.bfloat16)
    return xa, wa, oa, xr, wr, orr


@pytest.mark.parametrize("T", [2, 4, 8])
def test_c4_no_tail_local_group(T):
    S, K, N = 2048, 1024, 2048
    xa, wa, oa, xr, wr, orr = _tensors(T, S, K, N, True)
    comm = tpf.Communicator.local_group(T, max(tpf.sym_bytes_ag(T, 1, S, K, N // T), tpf.sym_bytes_rs(T, 1, S, K // T, N)))
    summ = _traced(comm, lambda: comm.ag_gemm(xa, wa, oa))
    assert len(summ) == T and trace.no_tail(summ), {r: v["tail_us"] for r, v in summ.items()}
    for kind in _kinds(T):
        for wire in (tpf.BF16, tpf.F32):
            summ = _traced(comm, lambda: comm.gemm_rs(xr, wr, orr, kind=kind, wire=wire))
            assert len(summ) == T and trace.no_tail(summ), (kind, wire, {r: v["tail_us"] for r, v in summ.items()})
    comm.close()


@pytest.mark.parametrize("T", [2, 4, 8])
def test_c4_no_tail_split_group(T):
    """Per-rank launch path: each rank's own communicator traces its own records."""
    S, K, N = 2048, 1024, 2048
    xa, wa, oa, xr, wr, orr = _tensors(T, S, K, N, True)
    comms = tpf.Communicator.split_group(T, max(tpf.sym_bytes_ag(T, 1, S, K, N // T), tpf.sym_bytes_rs(T, 1, S, K // T, N)))
    calls = [("ag", None)] + [("rs", k) for k in _kinds(T)]
    for op, kind in calls:
        def run():
            for r in range(T):
                if op == "ag":
                    comms[r].ag_gemm(xa[r], wa[r], oa[r])
                else:
                    comms[r].gemm_rs(xr[r], wr[r], orr[r], kind=kind)
        for _ in range(2):
            run()
        for c in comms:
            c.sync()
        bufs = [trace.alloc(100000) for _ in range(T)]
        for c, b in zip(comms, bufs):
            c.set_trace(b)
        run()
        for c in comms:
            c.sync()
            c.set_trace(None)
        for r, b in enumerate(bufs):
            summ = trace.summarize(trace.decode(b))
            assert list(summ) == [r] and trace.no_tail(summ), (op, kind, r, summ[r]["tail_us"])
    for c in comms:
        c.close()


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3"])
@pytest.mark.parametrize("T", [2, 4, 8])
def test_c4_no_tail_per_gpu_virtual(cfg, T):
    """One GPU of a TP group at full per-rank scale (virtual peers)."""
    S, K_ag, N_ag, K_rs, N_rs = {"cfg2": (8192, 4096, 28672, 14336, 4096),
                                 "cfg3": (16384, 8192, 10240, 8192, 8192)}[cfg]
    g = torch.Generator(device=DEV).manual_seed(0)
    x = torch.randn((1, S // T, K_ag), device=DEV, generator=g).to(torch.bfloat16)
    w = (torch.randn((K_ag, N_ag // T), device=DEV, generator=g) / 64).to(torch.bfloat16)
    y = torch.empty((1, S, N_ag // T), device=DEV, dtype=torch.bfloat16)
    xr = torch.randn((1, S, K_rs // T), device=DEV, generator=g).to(torch.bfloat16)
    wr = (torch.randn((K_rs // T, N_rs), device=DEV, generator=g) / 64).to(torch.bfloat16)
    yr = torch.empty((1, S // T, N_rs), device=DEV, dtype=torch.bfloat16)
    comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, K_ag, N_ag // T),
                                                 tpf.sym_bytes_rs(T, 1, S, K_rs // T, N_rs, 1, tpf.BF16)))
    summ = _traced(comm, lambda: comm.ag_gemm(x, w, y))
    assert trace.no_tail(summ), summ[0]["tail_us"]
    for kind in _kinds(T):
        summ = _traced(comm, lambda: comm.gemm_rs(xr, wr, yr, kind=kind, wire=tpf.BF16))
        assert trace.no_tail(summ), (kind, summ[0]["tail_us"])
    comm.close()


def _per_call_us(fn, n=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / n


def _fused_and_plain_us(fused, plain, rounds=5):
    """Best of `rounds` alternating rounds for each: on these power-capped GPUs the clock moves
    with temperature, and the fused op (more memory traffic) slows more as the GPU heats, so each
    side is taken at its best state of the same stretch of time."""
    for _ in range(3):
        fused()
        plain()
    torch.cuda.synchronize()
    f, g = [], []
    for _ in range(rounds):
        f.append(_per_call_us(fused))
        g.append(_per_call_us(plain))
    return min(f), min(g)


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3"])
def test_c6_fused_within_125pct_of_plain_gemm_per_gpu(cfg):
    """acceptance C6 analogue at TP = 8: fused op <= 1.25 x the plain per-rank GEMM."""
    T = 8
    S, K_ag, N_ag, K_rs, N_rs = {"cfg2": (8192, 4096, 28672, 14336, 4096),
                                 "cfg3": (16384, 8192, 10240, 8192, 8192)}[cfg]
    g = torch.Generator(device=DEV).manual_seed(1)
    x = torch.randn((1, S // T, K_ag), device=DEV, generator=g).to(torch.bfloat16)
    xg = torch.randn((1, S, K_ag), device=DEV, generator=g).to(torch.bfloat16)
    w = (torch.randn((K_ag, N_ag // T), device=DEV, generator=g) / 64).to(torch.bfloat16)
    y = torch.empty((1, S, N_ag // T), device=DEV, dtype=torch.bfloat16)
    xr = torch.randn((1, S, K_rs // T), device=DEV, generator=g).to(torch.bfloat16)
    wr = (torch.randn((K_rs // T, N_rs), device=DEV, generator=g) / 64).to(torch.bfloat16)
    yr = torch.empty((1, S // T, N_rs), device=DEV, dtype=torch.bfloat16)
    yg = torch.empty((1, S, N_rs), device=DEV, dtype=torch.bfloat16)
    comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, K_ag, N_ag // T),
                                                 tpf.sym_bytes_rs(T, 1, S, K_rs // T, N_rs, 1, tpf.BF16)))
    one = tpf.Communicator.create(0, 1, 0)
    ag, p_ag = _fused_and_plain_us(lambda: comm.ag_gemm(x, w, y), lambda: one.ag_gemm(xg, w, y))
    rs, p_rs = _fused_and_plain_us(lambda: comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=tpf.BF16),
                                   lambda: one.gemm_rs(xr, wr, yg))
    comm.sync()
    comm.close()
    one.close()
    print(f"{cfg} TP8 per GPU: AG {ag:.1f} us vs plain {p_ag:.1f} ({ag / p_ag:.3f}); "
          f"RS {rs:.1f} us vs plain {p_rs:.1f} ({rs / p_rs:.3f})")
    assert ag <= 1.25 * p_ag and rs <= 1.25 * p_rs
