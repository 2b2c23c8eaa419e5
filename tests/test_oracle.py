"""Pin the CPU oracle (oracle/tpf_oracle.c) before trusting it.

1. Against the golden vectors the reference's own tests hold
   (collectives_test.cpp:54-114,249-268; tensor_test.cpp:207-214).
2. Against the golden fixtures dumped from the compiled reference
   (tests/golden/make_golden.py).
3. Against the compiled reference itself on fresh random non-integer fp64 data
   (bit-exact: the restatement reproduces the reference's reduction order),
   when oracle/_ref is present.
"""
import json
import os

import numpy as np
import pytest

from oracle_lib import CIRCULAR, PAIRWISE, RING, Oracle, OracleError, Reference, have_reference

HERE = os.path.dirname(os.path.abspath(__file__))
O = Oracle()
KINDS = (RING, PAIRWISE, CIRCULAR)


def golden():
    with open(os.path.join(HERE, "golden", "schedules.json")) as f:
        return json.load(f)


# ------------------------------------------------- reference test known answers
def test_randint_golden_seed42():
    # tensor_test.cpp:207-214
    assert O.randint((1, 2, 2), 0, 8, 42).reshape(-1).tolist() == [6.0, 0.0, 2.0, 6.0]


def test_randint_degenerate_and_rejects():
    assert not O.randint((2, 2, 2), 0, 1, 9).any()
    with pytest.raises(OracleError):
        O.randint((1, 1, 1), 3, 3, 0)


def test_ring_index_formulas():
    # collectives_test.cpp:54-86
    assert O.ring_indices(False, 0, 1, 4) == (1, 3, 3)
    assert O.ring_indices(True, 0, 0, 4) == (1, 3, 3)
    assert O.ring_indices(False, 0, 0, 1) == (0, 0, 0)
    for n in range(1, 9):
        for r in range(n):
            assert O.ring_indices(False, r, 0, n)[2] == r          # AG: own slice first
            assert O.ring_indices(True, r, n - 1, n)[2] == r       # RS: own slice last
            assert sorted(O.ring_indices(False, r, i, n)[2] for i in range(n)) == list(range(n))
    with pytest.raises(OracleError):
        O.ring_indices(True, 4, 0, 4)


def test_pairwise_rounds_n4():
    # collectives_test.cpp:106-114: rounds {(0,1),(2,3)}, {(0,2),(1,3)}, {(0,3),(1,2)}
    t = O.schedule(PAIRWISE, 4)
    assert t[:, :3, 0].T.tolist() == [[1, 0, 3, 2], [2, 3, 0, 1], [3, 2, 1, 0]]


def test_schedule_rejections():
    with pytest.raises(OracleError):
        O.schedule(PAIRWISE, 3)
    with pytest.raises(OracleError):
        O.schedule(RING, 0)
    assert O.schedule(PAIRWISE, 1).size == 0


@pytest.mark.parametrize("kind", KINDS)
def test_corrupted_tables_rejected(kind):
    # collectives_test.cpp:152-160: a table with a wrong final slice fails check_schedule
    t = O.schedule(kind, 4).copy()
    assert O.check_schedule(kind, t)
    t[1, 3, 2] = 0
    assert not O.check_schedule(kind, t)
    t = O.schedule(kind, 4).copy()
    t[2, 0, 0] = -1
    assert not O.check_schedule(kind, t)


def test_indexed_sum_all_schedules():
    # collectives_test.cpp:249-268: entry(r,s) = 10r+s  => rank s holds 60+4s
    t = 4
    inputs = np.array([[[[10.0 * r + s] for s in range(4)]] for r in range(t)])
    for kind in KINDS:
        out = O.fuse_rs_identity(t, kind, 1, inputs)
        assert out[:, 0, 0, 0].tolist() == [60.0 + 4 * s for s in range(t)]


# ----------------------------------------------------------- golden fixtures
def test_schedules_match_golden():
    g = golden()
    for n in range(1, 9):
        for kind in KINDS:
            want = g["schedules"][f"{kind}/{n}"]
            if isinstance(want, dict):
                with pytest.raises(OracleError):
                    O.schedule(kind, n)
            else:
                got = O.schedule(kind, n)
                assert got.reshape(-1).tolist() == np.array(want, np.int32).reshape(-1).tolist(), (kind, n)
        for r in range(n):
            for i in range(n):
                assert list(O.ring_indices(False, r, i, n)) == g["ring_indices_ag"][str(n)][r][i]
                assert list(O.ring_indices(True, r, i, n)) == g["ring_indices_rs"][str(n)][r][i]
    assert O.randint((1, 2, 2), 0, 8, 42).reshape(-1).tolist() == g["randint_fill_1_2_2_0_8_42"]


def _cases():
    z = np.load(os.path.join(HERE, "golden", "cases.npz"))
    tags = sorted({k.split("/")[0] for k in z.files})
    return z, tags


def test_layer_outputs_match_golden():
    z, tags = _cases()
    assert tags
    for tag in tags:
        t, kind, m = (int(tag.split("_")[i][1:]) for i in range(3))
        x, up, down, x2, w2 = (z[f"{tag}/{k}"] for k in ("x", "up", "down", "x2", "w2"))
        assert np.array_equal(O.mlp_square(t, kind, m, x, up, down), z[f"{tag}/mlp"]), tag
        assert np.array_equal(O.column_parallel(t, m, x, up), z[f"{tag}/col"]), tag
        assert np.array_equal(O.row_parallel(t, kind, m, x2, w2), z[f"{tag}/row"]), tag


def test_golden_inputs_follow_reference_recipe():
    # the fixtures' inputs are reproducible with the oracle's randint + mix_seed
    z, tags = _cases()
    tag = tags[0]
    idx = 0
    x = O.randint(z[f"{tag}/x"].shape, 0, 5, O.mix_seed(idx % 5, 0))
    assert np.array_equal(x, z[f"{tag}/x"])


# ------------------------------------------------- live compiled reference
needs_ref = pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
@pytest.mark.parametrize("t", [1, 2, 4, 8])
def test_restatement_bitexact_vs_reference_random(t):
    R = Reference()
    rng = np.random.default_rng(t)
    for kind in KINDS:
        if kind == PAIRWISE and t % 2 and t != 1:
            continue
        for m in ((1, 2) if kind == RING else (1,)):
            b, s, k, n = 2, 32, 16, 8
            x = rng.uniform(-1, 1, (b, s, k)) * 10.0 ** rng.integers(-3, 3)
            w = rng.uniform(-1, 1, (k, n))
            assert np.array_equal(R.row_parallel(t, kind, m, x, w), O.row_parallel(t, kind, m, x, w))
            assert np.array_equal(R.column_parallel(t, m, x, w), O.column_parallel(t, m, x, w))
            inp = rng.uniform(-1, 1, (t, b, s, k))
            assert np.array_equal(R.fuse_rs_identity(t, kind, m, inp), O.fuse_rs_identity(t, kind, m, inp))


@needs_ref
def test_reference_rejections_match():
    R = Reference()
    x = np.zeros((1, 6, 4))
    w = np.zeros((4, 4))
    for args in [(4, RING, 1), (2, RING, 2), (2, PAIRWISE, 2)]:  # S % (T*m) != 0, pairwise m>1
        with pytest.raises(OracleError):
            R.row_parallel(*args, x, w)
        with pytest.raises(OracleError):
            O.row_parallel(*args, x, w)


@needs_ref
@pytest.mark.parametrize("t", [1, 2, 4])
def test_attention_a2a_restatement_bitexact(t):
    """UP (Alg. 5, fuse_all_to_all_attention): restatement == compiled reference."""
    R = Reference()
    rng = np.random.default_rng(40 + t)
    for heads in (1, 2):
        b, s, dh = 2, 8 * t, 4
        q, k, v = (rng.uniform(-1, 1, (t, b * heads, s, dh)) for _ in range(3))
        for scale in (True, False):
            assert np.array_equal(O.attention_a2a(t, b, heads, q, k, v, scale),
                                  R.attention_a2a(t, b, heads, q, k, v, scale))


@needs_ref
@pytest.mark.parametrize("t", [1, 2, 4])
def test_query_split_attention_restatement_bitexact(t):
    """Alg. 4 (query_split_attention): restatement == compiled reference, every schedule."""
    R = Reference()
    rng = np.random.default_rng(60 + t)
    b, heads, s, dh, d = 2, 2, 8 * t, 4, 8
    q, k, v = (rng.uniform(-1, 1, (t, b * heads, s, dh)) for _ in range(3))
    w_o = rng.uniform(-1, 1, (t * heads * dh, d))
    for kind in KINDS:
        if kind == PAIRWISE and t % 2 and t != 1:
            continue
        assert np.array_equal(O.query_split_attention(t, kind, b, heads, q, k, v, w_o),
                              R.query_split_attention(t, kind, b, heads, q, k, v, w_o))


@needs_ref
@pytest.mark.parametrize("t", [1, 2, 4])
def test_ulysses_a2a_restatement_bitexact(t):
    """Ulysses first all-to-all (layers_test.cpp:347-397 drive of ref_all_to_all): restatement
    == compiled reference, and it reproduces the direct head-group layout."""
    R = Reference()
    rng = np.random.default_rng(90 + t)
    b, heads, sl, dh = 2, 2 * t, 3, 4
    x = rng.uniform(-1, 1, (t, b * heads, sl, dh))
    got = O.ulysses_a2a(t, b, heads, x)
    assert np.array_equal(got, R.ulysses_a2a(t, b, heads, x))
    full = x.reshape(t, b, heads, sl, dh).transpose(1, 2, 0, 3, 4).reshape(b, heads, t * sl, dh)
    hl = heads // t
    for g in range(t):
        assert np.array_equal(got[g], full[:, g * hl:(g + 1) * hl].reshape(b * hl, t * sl, dh))


def test_ulysses_a2a_rejects_indivisible():
    with pytest.raises(OracleError):
        O.ulysses_a2a(3, 1, 4, np.zeros((3, 4, 2, 4)))
