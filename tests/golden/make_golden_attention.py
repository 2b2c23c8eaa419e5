"""Generate tests/golden/attention.npz from the REFERENCE ITSELF (SPEC acceptance C2 analogue).

Runs the unmodified reference (oracle/_ref/libtpfuse_ref.so, compiled by oracle/Makefile from
/root/reference/proj/src) on the acceptance suite's attention data recipe -- the exact lattice
k/8 in [-1, 1) (real_fill / real_matrix, experiment.cpp:195-205), exactly representable in bf16
-- and freezes its fuse_all_to_all_attention (layers.cpp:174-218) and query_split_attention
(layers.cpp:149-172) outputs (float16: the GPU tolerance is 2e-2) for
tests/test_gpu_attention_golden.py. Shapes use head_dim 128 and 128-row slices (the fused
tcgen05 attention kernel's shape). Only outputs are stored: the test regenerates the inputs with
the oracle's randint, asserted here to equal the reference's randint_fill on every input.

    python tests/golden/make_golden_attention.py      # in the build container
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Oracle, Reference  # noqa: E402

DH = 128
UP_CASES = [(2, 2), (4, 1)]                       # (T, heads per rank), batch 1
QS_CASES = [(2, 1, 256, (0, 1, 2)), (4, 1, 256, (0,))]  # (T, heads per rank, D, schedules)


def up_inputs(gen, T, heads):
    S = 128 * T
    return [gen.randint((T * heads, S, DH), -8, 8, Oracle().mix_seed(T, salt)) for salt in (10, 11, 12)]


def qs_inputs(gen, T, heads, D, matrix):
    S = 128 * T
    qkv = [gen.randint((T * heads, S, DH), -8, 8, Oracle().mix_seed(T, salt)) for salt in (20, 21, 22)]
    return qkv + [matrix(T * heads * DH, D, -8, 8, Oracle().mix_seed(T, 23))]


def main() -> None:
    R, O = Reference(), Oracle()
    arrays = {}
    for T, heads in UP_CASES:
        ins = up_inputs(R, T, heads)
        assert all(np.array_equal(a, b) for a, b in zip(ins, up_inputs(O, T, heads)))
        f = [a.astype(np.float64).reshape(T, heads, 128 * T, DH) / 8 for a in ins]
        arrays[f"up_t{T}_h{heads}"] = R.attention_a2a(T, 1, heads, *f, True).astype(np.float16)
    for T, heads, D, kinds in QS_CASES:
        ins = qs_inputs(R, T, heads, D, R.randint_matrix)
        o_matrix = lambda r, c, lo, hi, seed: O.randint((r, c), lo, hi, seed)  # noqa: E731
        assert all(np.array_equal(a, b) for a, b in zip(ins, qs_inputs(O, T, heads, D, o_matrix)))
        f = [a.astype(np.float64).reshape(T, heads, 128 * T, DH) / 8 for a in ins[:3]]
        w_o = ins[3].astype(np.float64) / 128  # a 1/128 lattice keeps the projection in range
        for kind in kinds:
            arrays[f"qs_t{T}_k{kind}"] = R.query_split_attention(T, kind, 1, heads, *f, w_o, True).astype(np.float16)
    np.savez_compressed(os.path.join(HERE, "attention.npz"), **arrays)
    print("wrote", sorted(arrays))


if __name__ == "__main__":
    main()
