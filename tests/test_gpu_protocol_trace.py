"""The reference's protocol-order tests, checked on the kernel's own device timeline.

collectives_test.cpp asserts properties of the order in which the fused collectives compute and
communicate, by instrumenting the compute function and the fabric:
  * FuseAllGather.OwnSliceComputedFirst (:212-237): iteration 0 computes the rank's own slice;
  * FuseReduceScatter.OwnSliceComputedLast (:326-356): the final iteration computes the own slice;
  * FuseReduceScatter.NoCommunicationPostedInFinalIteration (:311-324);
  * FuseAllToAllAttention.PostsExactlyGroupMinusOneTransfers (layers_test.cpp:399-412) -- for the
    GEMM collectives: every rank sends in exactly T - 1 iterations.
Here the same properties are read from the %globaltimer records the fused kernel writes
(paper_2604_24013_b200.trace) with the schedule the launch used, per rank, in the local group.
"""
import pytest
import torch

import paper_2604_24013_b200 as tpf
from paper_2604_24013_b200 import trace

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def _run_traced(comm, call):
    call()
    comm.sync()
    buf = trace.alloc(300000)
    comm.set_trace(buf)
    call()
    comm.sync()
    comm.set_trace(None)
    return trace.decode(buf)


def _kinds(T):
    return [tpf.RING, tpf.CIRCULAR] + ([tpf.PAIRWISE] if T % 2 == 0 else [])


@pytest.mark.parametrize("T", [2, 4, 8])
def test_rs_sends_in_exactly_t_minus_1_iterations_and_not_in_the_last(T):
    S, K, N = 2048, 512, 1024
    g = torch.Generator(device=DEV).manual_seed(T)
    x = torch.randn((T, 1, S, K // T), device=DEV, generator=g).to(torch.bfloat16)
    w = (torch.randn((T, K // T, N), device=DEV, generator=g) / 16).to(torch.bfloat16)
    y = torch.empty((T, 1, S // T, N), device=DEV, dtype=torch.bfloat16)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_rs(T, 1, S, K // T, N))
    for kind in _kinds(T):
        recs = _run_traced(comm, lambda: comm.gemm_rs(x, w, y, kind=kind))
        sched = tpf.build_schedule(kind, T)
        for r in range(T):
            flags = [q for q in recs if q.rank == r and q.kind == trace.TR_FLAG]
            tiles = [q for q in recs if q.rank == r and q.kind == trace.TR_TILE]
            # NoCommunicationPostedInFinalIteration + exactly T - 1 sending iterations
            assert sorted({q.step for q in flags}) == list(range(T - 1)), (kind, r)
            assert sorted({q.step for q in tiles}) == list(range(T)), (kind, r)
            # OwnSliceComputedLast: the schedule's final iteration is the own slice (an
            # iteration-order property in the reference). On the timeline, each final-step tile
            # ends after every transfer it consumes was posted: the predecessor's step T-2
            # running sum (pipelined) or all T-1 partners' partials (pairwise). (Not after this
            # rank's own step T-2 tiles: those feed another rank and run in the same round on
            # other CTA pairs, so they may end slightly later.)
            assert sched[r][T - 1] == (-1, -1, r)
            per_step = len({q.index for q in tiles if q.step == 0})  # (several records per tile)
            assert {q.index for q in tiles} == set(range(T * per_step)), (kind, r)
            consumed = range(T - 1) if kind == tpf.PAIRWISE else [T - 2]
            for tile in range(per_step):
                end = max(q.t1 for q in tiles if q.step == T - 1 and q.index % per_step == tile)
                for s in consumed:
                    src = sched[r][s][1]
                    posted = [q.t1 for q in recs if q.rank == src and q.kind == trace.TR_FLAG and q.step == s
                              and q.index % per_step == tile]
                    assert posted and max(posted) <= end, (kind, r, tile, s, src)
            # every transfer is published before the rank's last tile ends (no tail)
            assert max(q.t1 for q in flags) <= max(q.t1 for q in tiles), (kind, r)
    comm.close()


@pytest.mark.parametrize("T", [2, 4, 8])
def test_ag_forwards_in_exactly_t_minus_1_steps_own_slice_first(T):
    S, K, N = 2048, 1024, 2048
    g = torch.Generator(device=DEV).manual_seed(10 + T)
    x = torch.randn((T, 1, S // T, K), device=DEV, generator=g).to(torch.bfloat16)
    w = (torch.randn((T, K, N // T), device=DEV, generator=g) / 32).to(torch.bfloat16)
    y = torch.empty((T, 1, S, N // T), device=DEV, dtype=torch.bfloat16)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ag(T, 1, S, K, N // T))
    recs = _run_traced(comm, lambda: comm.ag_gemm(x, w, y))
    for r in range(T):
        pieces = [q for q in recs if q.rank == r and q.kind == trace.TR_AG_PIECE]
        loops = [q for q in recs if q.rank == r and q.kind == trace.TR_MAINLOOP]
        # the ring forwards in T - 1 steps (slots 0 .. T-2), the last step forwards nothing
        assert sorted({q.step for q in pieces}) == list(range(T - 1)), r
        # OwnSliceComputedFirst: iteration 0 computes the own slice (ring_indices_ag), and the
        # first main loop on the timeline is an iteration-0 tile
        assert tpf.ring_indices_ag(r, 0, T)[2] == r
        assert min(loops, key=lambda q: q.t0).step == 0, r
        # iteration 0 reads only local data: no producer ever waited on a wire image for it
        assert not [q for q in recs if q.rank == r and q.kind == trace.TR_WAIT_A and q.step == 0], r
    comm.close()
