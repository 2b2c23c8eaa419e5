"""Product schedule module (libtpfuse_b200 host C++, via the C ABI) — CPU only.

Bit-exact with the reference's build_schedule / ring_indices_* (golden tables
dumped from the compiled reference) and with the same rejections / exception
types (collectives_test.cpp:54-160, SPEC acceptance C3)."""
import json
import os

import pytest

import paper_2604_24013_b200 as tpf

HERE = os.path.dirname(os.path.abspath(__file__))
KINDS = (tpf.RING, tpf.PAIRWISE, tpf.CIRCULAR)


def golden():
    with open(os.path.join(HERE, "golden", "schedules.json")) as f:
        return json.load(f)


def test_tables_bitexact_with_reference_golden():
    g = golden()
    for n in range(1, 9):
        for kind in KINDS:
            want = g["schedules"][f"{kind}/{n}"]
            if isinstance(want, dict):
                with pytest.raises(ValueError, match="even rank count"):
                    tpf.build_schedule(kind, n)
                continue
            got = tpf.build_schedule(kind, n)
            if n == 1:
                assert got == [[]]
            else:
                assert [[list(st) for st in row] for row in got] == want, (kind, n)
        for r in range(n):
            for i in range(n):
                assert list(tpf.ring_indices_ag(r, i, n)) == g["ring_indices_ag"][str(n)][r][i]
                assert list(tpf.ring_indices_rs(r, i, n)) == g["ring_indices_rs"][str(n)][r][i]


def test_appendix_a_examples():
    ring = tpf.build_schedule(tpf.RING, 4)
    assert ring[0] == [(1, 3, 3), (1, 3, 2), (1, 3, 1), (-1, -1, 0)]
    circ = tpf.build_schedule(tpf.CIRCULAR, 4)
    assert circ[1] == [(0, 2, 2), (0, 2, 3), (0, 2, 0), (-1, -1, 1)]
    pw8 = tpf.build_schedule(tpf.PAIRWISE, 8)
    assert [st[2] for st in pw8[0]] == [5, 3, 1, 6, 4, 2, 7, 0]  # SURVEY App. A (rounds, then own)


@pytest.mark.parametrize("n", [2, 4, 6, 8, 3, 5, 7])
def test_invariants_hold(n):
    # SPEC acceptance C3: n-1 sends / recvs, own slice last, pairwise disjoint rounds
    for kind in KINDS:
        if kind == tpf.PAIRWISE and n % 2:
            continue
        steps = tpf.build_schedule(kind, n)
        tpf.check_schedule(kind, steps)
        for r, row in enumerate(steps):
            assert sum(st[0] >= 0 for st in row) == n - 1
            assert sum(st[1] >= 0 for st in row) == n - 1
            assert row[-1] == (-1, -1, r)
        if kind == tpf.PAIRWISE:
            for i in range(n - 1):
                partners = [steps[r][i][0] for r in range(n)]
                assert all(partners[partners[r]] == r for r in range(n))


def test_ring_final_iteration_has_no_comm():
    # collectives_test.cpp:311-324 analogue on the table: nothing posted in iteration n-1
    for n in (2, 4, 8):
        for kind in KINDS:
            for row in tpf.build_schedule(kind, n):
                assert row[-1][0] == -1 and row[-1][1] == -1


@pytest.mark.parametrize("kind", KINDS)
def test_corrupted_table_rejected(kind):
    steps = [list(map(list, row)) for row in tpf.build_schedule(kind, 4)]
    steps[1][3][2] = 0  # own slice no longer last
    with pytest.raises(tpf.LogicError, match="check_schedule"):
        tpf.check_schedule(kind, steps)
    steps = [list(map(list, row)) for row in tpf.build_schedule(kind, 4)]
    steps[0][0] = [-1, -1, steps[0][0][2]]  # a send dropped
    with pytest.raises(tpf.LogicError):
        tpf.check_schedule(kind, steps)


def test_duplicate_delivery_rejected():
    # exactly-once delivery (check_delivery): two ranks computing the same slice
    steps = [list(map(list, row)) for row in tpf.build_schedule(tpf.RING, 4)]
    steps[0][0][2], steps[0][1][2] = steps[0][1][2], steps[0][0][2]
    with pytest.raises(tpf.LogicError, match="exactly once|contributions"):
        tpf.check_schedule(tpf.RING, steps)


def test_argument_errors():
    with pytest.raises(ValueError, match="outside"):
        tpf.ring_indices_ag(4, 0, 4)
    with pytest.raises(ValueError):
        tpf.ring_indices_rs(0, -1, 4)
    with pytest.raises(ValueError, match="n must be >= 1"):
        tpf.build_schedule(tpf.RING, 0)
    assert tpf.ring_indices_ag(0, 0, 1) == (0, 0, 0)
    assert tpf.ring_indices_rs(0, 0, 1) == (0, 0, 0)
