"""ctypes loaders for the CPU oracle (TEST INFRASTRUCTURE ONLY).

* ``Oracle``    — oracle/liboracle.so, the plain-C restatement (tpf_oracle.c).
* ``Reference`` — oracle/_ref/libtpfuse_ref.so, the unmodified reference sources
  (/root/reference/proj/src) compiled in place plus the C-ABI bridge
  (ref_bridge.cpp). Optional: absent on a checkout where the reference was
  never mounted; tests that need it skip.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtpfuse_ref.so")

RING, PAIRWISE, CIRCULAR = 0, 1, 2
KIND_NAMES = {RING: "ring", PAIRWISE: "pairwise", CIRCULAR: "circular-slices"}

_D = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_I = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64 = C.c_int64


def _ensure_built(path: str) -> None:
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"),
                        os.path.join(ROOT, "oracle", "liboracle.so")], check=True)


class OracleError(RuntimeError):
    pass


class Oracle:
    """Plain-C restatement of the reference (fp64)."""

    def __init__(self) -> None:
        _ensure_built(ORACLE_SO)
        L = C.CDLL(ORACLE_SO)
        L.or_randint_fill.argtypes = [_i64, C.c_int, C.c_int, C.c_uint64, _D]
        L.or_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.or_mix_seed.restype = C.c_uint64
        L.or_ring_indices.argtypes = [C.c_int] * 4 + [_I]
        L.or_build_schedule.argtypes = [C.c_int, C.c_int, _I]
        L.or_check_schedule.argtypes = [C.c_int, C.c_int, _I]
        L.or_matmul.argtypes = [_i64, _i64, _i64, _D, _D, _D]
        L.or_column_parallel.argtypes = [C.c_int, C.c_int] + [_i64] * 4 + [_D, _D, _D]
        L.or_row_parallel.argtypes = [C.c_int] * 3 + [_i64] * 4 + [_D, _D, _D]
        L.or_fuse_rs_identity.argtypes = [C.c_int] * 3 + [_i64] * 3 + [_D, _D]
        L.or_mlp_square.argtypes = [C.c_int] * 3 + [_i64] * 4 + [_D, _D, _D, _D]
        L.or_attention_a2a.argtypes = [C.c_int] * 3 + [_i64] * 2 + [C.c_int, _D, _D, _D, _D]
        L.or_query_split_attention.argtypes = [C.c_int] * 4 + [_i64] * 3 + [C.c_int, _D, _D, _D, _D, _D]
        L.or_ulysses_a2a.argtypes = [C.c_int] * 3 + [_i64] * 2 + [_D, _D]
        self.L = L

    @staticmethod
    def _chk(rc: int, what: str) -> None:
        if rc != 0:
            raise OracleError(what)

    def randint(self, shape, lo, hi, seed) -> np.ndarray:
        out = np.empty(int(np.prod(shape)), np.float64)
        self._chk(self.L.or_randint_fill(out.size, lo, hi, seed, out), "randint_fill: empty range")
        return out.reshape(shape)

    def mix_seed(self, seed: int, salt: int) -> int:
        return int(self.L.or_mix_seed(seed, salt))

    def ring_indices(self, rs: bool, r: int, i: int, n: int):
        out = np.zeros(3, np.int32)
        self._chk(self.L.or_ring_indices(int(rs), r, i, n, out), "ring_indices: bad args")
        return tuple(int(v) for v in out)

    def schedule(self, kind: int, n: int) -> np.ndarray:
        out = np.zeros(max(n * n * 3, 1), np.int32)
        self._chk(self.L.or_build_schedule(kind, n, out), "build_schedule rejected")
        return out[: n * n * 3].reshape(n, n, 3) if n > 1 else np.zeros((1, 0, 3), np.int32)

    def check_schedule(self, kind: int, table: np.ndarray) -> bool:
        n = table.shape[0]
        t = np.ascontiguousarray(table, np.int32).reshape(-1)
        if t.size == 0:
            t = np.zeros(1, np.int32)
        return self.L.or_check_schedule(kind, n, t) == 0

    def matmul(self, x: np.ndarray, w: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        w = np.ascontiguousarray(w, np.float64)
        k, n = w.shape
        rows = x.size // k
        out = np.empty(rows * n, np.float64)
        self.L.or_matmul(rows, k, n, x.reshape(-1), w.reshape(-1), out)
        return out.reshape(x.shape[:-1] + (n,))

    def column_parallel(self, t, m, x_full, w_full):
        b, s, k = x_full.shape
        n = w_full.shape[1]
        out = np.empty(t * b * s * (n // t), np.float64)
        self._chk(self.L.or_column_parallel(t, m, b, s, k, n, np.ascontiguousarray(x_full).reshape(-1),
                                            np.ascontiguousarray(w_full).reshape(-1), out),
                  "column_parallel: invalid arguments")
        return out.reshape(t, b, s, n // t)

    def row_parallel(self, t, kind, m, x_full, w_full):
        b, s, k = x_full.shape
        n = w_full.shape[1]
        out = np.empty(b * s * n, np.float64)
        self._chk(self.L.or_row_parallel(t, kind, m, b, s, k, n, np.ascontiguousarray(x_full).reshape(-1),
                                         np.ascontiguousarray(w_full).reshape(-1), out),
                  "row_parallel: invalid arguments")
        return out.reshape(t, b, s // t, n)

    def fuse_rs_identity(self, t, kind, m, inputs):
        _, b, s, d = inputs.shape
        out = np.empty(b * s * d, np.float64)
        self._chk(self.L.or_fuse_rs_identity(t, kind, m, b, s, d, np.ascontiguousarray(inputs).reshape(-1), out),
                  "fuse_reduce_scatter: invalid arguments")
        return out.reshape(t, b, s // t, d)

    def mlp_square(self, t, kind, m, x_full, up, down):
        b, s, d = x_full.shape
        h = up.shape[1]
        out = np.empty(b * s * d, np.float64)
        self._chk(self.L.or_mlp_square(t, kind, m, b, s, d, h, np.ascontiguousarray(x_full).reshape(-1),
                                       np.ascontiguousarray(up).reshape(-1),
                                       np.ascontiguousarray(down).reshape(-1), out),
                  "tpsp_mlp_forward: invalid arguments")
        return out.reshape(t, b, s // t, d)


    def attention_a2a(self, t, batch, heads, q, k, v, scale=True):
        """q/k/v: (T, batch*heads, S, dh) -> (T, batch, S/T, T*heads*dh)."""
        _, bh, s, dh = q.shape
        out = np.empty(t * batch * (s // t) * t * heads * dh, np.float64)
        self._chk(self.L.or_attention_a2a(t, batch, heads, s, dh, int(scale), np.ascontiguousarray(q).reshape(-1),
                                          np.ascontiguousarray(k).reshape(-1), np.ascontiguousarray(v).reshape(-1),
                                          out), "fuse_all_to_all_attention: invalid arguments")
        return out.reshape(t, batch, s // t, t * heads * dh)


    def query_split_attention(self, t, kind, batch, heads, q, k, v, w_o, scale=True):
        """q/k/v: (T, batch*heads, S, dh); w_o: (T*heads*dh, d) -> (T, batch, S/T, d)."""
        _, bh, s, dh = q.shape
        d = w_o.shape[1]
        out = np.empty(t * batch * (s // t) * d, np.float64)
        self._chk(self.L.or_query_split_attention(t, kind, batch, heads, s, dh, d, int(scale),
                                                  np.ascontiguousarray(q).reshape(-1), np.ascontiguousarray(k).reshape(-1),
                                                  np.ascontiguousarray(v).reshape(-1),
                                                  np.ascontiguousarray(w_o).reshape(-1), out),
                  "query_split_attention: invalid arguments")
        return out.reshape(t, batch, s // t, d)


    def ulysses_a2a(self, t, batch, heads, x):
        """x: (T, batch*heads, S/T, dh) sequence-sharded -> (T, batch*heads/T, S, dh) head-sharded."""
        _, bh, sl, dh = x.shape
        out = np.empty(x.size, np.float64)
        self._chk(self.L.or_ulysses_a2a(t, batch, heads, sl * t, dh, np.ascontiguousarray(x, np.float64).reshape(-1), out), "ulysses_a2a: invalid arguments")
        return out.reshape(t, batch * heads // t, sl * t, dh)


def have_reference() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The reference library itself (compiled from /root/reference)."""

    def __init__(self) -> None:
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_schedule.argtypes = [C.c_int, C.c_int, _I]
        L.ref_ring_indices.argtypes = [C.c_int] * 4 + [_I]
        L.ref_randint_fill.argtypes = [_i64] * 3 + [C.c_int, C.c_int, C.c_uint64, _D]
        L.ref_randint_matrix.argtypes = [_i64] * 2 + [C.c_int, C.c_int, C.c_uint64, _D]
        L.ref_column_parallel.argtypes = [C.c_int, C.c_int] + [_i64] * 4 + [_D, _D, _D]
        L.ref_row_parallel.argtypes = [C.c_int] * 3 + [_i64] * 4 + [_D, _D, _D]
        L.ref_fuse_rs_identity.argtypes = [C.c_int] * 3 + [_i64] * 3 + [_D, _D]
        L.ref_mlp_square.argtypes = [C.c_int] * 3 + [_i64] * 4 + [_D, _D, _D, _D]
        L.ref_time_ops.argtypes = [C.c_int] + [_i64] * 6 + [C.c_int, _D, _D]
        L.ref_attention_a2a.argtypes = [C.c_int] * 3 + [_i64] * 2 + [C.c_int, _D, _D, _D, _D]
        L.ref_query_split_attention.argtypes = [C.c_int] * 4 + [_i64] * 3 + [C.c_int, _D, _D, _D, _D, _D]
        L.ref_ulysses_a2a.argtypes = [C.c_int] * 3 + [_i64] * 2 + [_D, _D]
        self.L = L

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(self.L.ref_last_error().decode())

    def schedule(self, kind, n):
        out = np.zeros(max(n * n * 3, 1), np.int32)
        self._chk(self.L.ref_build_schedule(kind, n, out))
        return out[: n * n * 3].reshape(n, n, 3) if n > 1 else np.zeros((1, 0, 3), np.int32)

    def ring_indices(self, rs, r, i, n):
        out = np.zeros(3, np.int32)
        self._chk(self.L.ref_ring_indices(int(rs), r, i, n, out))
        return tuple(int(v) for v in out)

    def randint(self, shape, lo, hi, seed):
        b, s, d = shape
        out = np.empty(b * s * d, np.float64)
        self._chk(self.L.ref_randint_fill(b, s, d, lo, hi, seed, out))
        return out.reshape(shape)

    def randint_matrix(self, rows, cols, lo, hi, seed):
        out = np.empty(rows * cols, np.float64)
        self._chk(self.L.ref_randint_matrix(rows, cols, lo, hi, seed, out))
        return out.reshape(rows, cols)

    def column_parallel(self, t, m, x_full, w_full):
        b, s, k = x_full.shape
        n = w_full.shape[1]
        out = np.empty(t * b * s * (n // t), np.float64)
        self._chk(self.L.ref_column_parallel(t, m, b, s, k, n, np.ascontiguousarray(x_full).reshape(-1),
                                             np.ascontiguousarray(w_full).reshape(-1), out))
        return out.reshape(t, b, s, n // t)

    def row_parallel(self, t, kind, m, x_full, w_full):
        b, s, k = x_full.shape
        n = w_full.shape[1]
        out = np.empty(b * s * n, np.float64)
        self._chk(self.L.ref_row_parallel(t, kind, m, b, s, k, n, np.ascontiguousarray(x_full).reshape(-1),
                                          np.ascontiguousarray(w_full).reshape(-1), out))
        return out.reshape(t, b, s // t, n)

    def fuse_rs_identity(self, t, kind, m, inputs):
        _, b, s, d = inputs.shape
        out = np.empty(b * s * d, np.float64)
        self._chk(self.L.ref_fuse_rs_identity(t, kind, m, b, s, d, np.ascontiguousarray(inputs).reshape(-1), out))
        return out.reshape(t, b, s // t, d)

    def mlp_square(self, t, kind, m, x_full, up, down):
        b, s, d = x_full.shape
        h = up.shape[1]
        out = np.empty(b * s * d, np.float64)
        self._chk(self.L.ref_mlp_square(t, kind, m, b, s, d, h, np.ascontiguousarray(x_full).reshape(-1),
                                        np.ascontiguousarray(up).reshape(-1),
                                        np.ascontiguousarray(down).reshape(-1), out))
        return out.reshape(t, b, s // t, d)

    def attention_a2a(self, t, batch, heads, q, k, v, scale=True):
        _, bh, s, dh = q.shape
        out = np.empty(t * batch * (s // t) * t * heads * dh, np.float64)
        self._chk(self.L.ref_attention_a2a(t, batch, heads, s, dh, int(scale), np.ascontiguousarray(q).reshape(-1),
                                           np.ascontiguousarray(k).reshape(-1), np.ascontiguousarray(v).reshape(-1),
                                           out))
        return out.reshape(t, batch, s // t, t * heads * dh)

    def query_split_attention(self, t, kind, batch, heads, q, k, v, w_o, scale=True):
        _, bh, s, dh = q.shape
        d = w_o.shape[1]
        out = np.empty(t * batch * (s // t) * d, np.float64)
        self._chk(self.L.ref_query_split_attention(t, kind, batch, heads, s, dh, d, int(scale),
                                                   np.ascontiguousarray(q).reshape(-1), np.ascontiguousarray(k).reshape(-1),
                                                   np.ascontiguousarray(v).reshape(-1),
                                                   np.ascontiguousarray(w_o).reshape(-1), out))
        return out.reshape(t, batch, s // t, d)

    def ulysses_a2a(self, t, batch, heads, x):
        """x: (T, batch*heads, S/T, dh) sequence-sharded -> (T, batch*heads/T, S, dh) head-sharded."""
        _, bh, sl, dh = x.shape
        out = np.empty(x.size, np.float64)
        self._chk(self.L.ref_ulysses_a2a(t, batch, heads, sl * t, dh, np.ascontiguousarray(x, np.float64).reshape(-1), out))
        return out.reshape(t, batch * heads // t, sl * t, dh)

    def time_ops(self, t, b, s, k_ag, n_ag, k_rs, n_rs, reps=1):
        """Per-repetition wall seconds of the reference's AG-GEMM and GEMM-RS."""
        ag = np.zeros(reps, np.float64)
        rs = np.zeros(reps, np.float64)
        self._chk(self.L.ref_time_ops(t, b, s, k_ag, n_ag, k_rs, n_rs, reps, ag, rs))
        return ag.tolist(), rs.tolist()

    def bench_csv(self, layer="mlp", tp=4, batch=2, seq=64, d_model=32, heads=4, granularity=1,
                  schedule="ring", seed=0, reps=2) -> str:
        """The reference's own run_bench CSV text (experiment.cpp:842-860) for a small config."""
        buf = C.create_string_buffer(1 << 16)
        self.L.ref_bench_csv.argtypes = [C.c_char_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                         C.c_char_p, C.c_uint64, C.c_int, C.c_char_p, C.c_int64]
        self._chk(self.L.ref_bench_csv(layer.encode(), tp, batch, seq, d_model, heads, granularity,
                                       schedule.encode(), seed, reps, buf, len(buf)))
        return buf.value.decode()
