"""Randomized (fixed-seed) shape / schedule / granularity sweep of the two fused
collectives against the oracle, on integer data (the reference's exact recipe), so every
case must be bit-exact: GPU fp32 accumulation and fp32 wire are exact on these values.
Covers odd group sizes, ragged chunks (rows not a multiple of 128), K / N not multiples
of the tile sizes, B > 1 and m > 1."""
import numpy as np
import pytest

import paper_2604_24013_b200 as tpf
from test_gpu_parity import O, run_ag, run_rs

pytestmark = pytest.mark.gpu


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


@pytest.mark.parametrize("T,kind,m,B,S,K,N", _cases(24, 2026, "rs"))
def test_fuzz_gemm_rs_exact(T, kind, m, B, S, K, N):
    x = O.randint((B, S, K), 0, 5, 11 + S)
    w = O.randint((K, N), -2, 2, 12 + N)
    got = run_rs(T, kind, m, x, w)
    assert np.array_equal(got, O.row_parallel(T, kind, m, x, w))


@pytest.mark.parametrize("T,kind,m,B,S,K,N", _cases(24, 2027, "ag"))
def test_fuzz_ag_gemm_exact(T, kind, m, B, S, K, N):
    x = O.randint((B, S, K), 0, 5, 13 + S)
    w = O.randint((K, N), -2, 2, 14 + N)
    got = run_ag(T, m, x, w)
    assert np.array_equal(got, O.column_parallel(T, m, x, w))
