"""B200-native CommFuse hot path (arXiv 2604.24013): fused AG-GEMM / GEMM-RS, the DP
gradient / parameter collectives, and the fused attention all-to-alls (Ulysses, query-split).

Python host mirror of the reference's operator API for this path
(/root/reference/proj/include/tpfuse/{collectives,layers}.hpp) over the C ABI
in include/tpf.h (libtpfuse_b200.so, built in-tree). torch is used only for
device memory, streams and torch.distributed plumbing.

There is no CPU or PyTorch fallback: if the shared library is missing, import
fails; if no sm_100 device is present, every data-path call raises TpfCudaError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
# TPF_LIB_PATH: an alternative build of the same library (dev A/B experiments only)
LIB_PATH = os.environ.get("TPF_LIB_PATH") or os.path.join(_HERE, "libtpfuse_b200.so")

RING, PAIRWISE, CIRCULAR = 0, 1, 2
KIND_NAMES = {RING: "ring", PAIRWISE: "pairwise", CIRCULAR: "circular-slices"}
BF16, F32 = 0, 1
ACT_NONE, ACT_SQUARE, ACT_SWIGLU = 0, 1, 2
IPC_HANDLE_BYTES = 64

# include/tpf.h error codes -> reference exception types (SURVEY §8(b) Errors)
E_INVALID, E_SHAPE, E_LOGIC, E_CUDA, E_PEER, E_CAPACITY = -1, -2, -3, -4, -5, -6


class ShapeError(ValueError):
    """tpfuse::ShapeError (a std::invalid_argument)."""


class LogicError(RuntimeError):
    """std::logic_error (check_schedule)."""


class GroupError(RuntimeError):
    """tpfuse::GroupError: a rank failed (here: peer flag wait timed out)."""


class TpfCudaError(RuntimeError):
    """CUDA failure or no sm_100 device."""


class CapacityError(RuntimeError):
    """Symmetric heap too small for the call."""


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not built: run `make -C {_HERE}` (or __graft_entry__.build()). "
        "There is no fallback path.")

_lib = C.CDLL(LIB_PATH)
_vp, _i64, _i32p = C.c_void_p, C.c_int64, C.POINTER(C.c_int32)
_lib.tpf_last_error.restype = C.c_char_p
_lib.tpf_ring_indices.argtypes = [C.c_int] * 4 + [_i32p]
_lib.tpf_schedule_build.argtypes = [C.c_int, C.c_int, _i32p]
_lib.tpf_schedule_check.argtypes = [C.c_int, C.c_int, _i32p]
_lib.tpf_comm_create.argtypes = [C.c_int, C.c_int, C.c_size_t, C.POINTER(_vp)]
_lib.tpf_comm_create_virtual.argtypes = [C.c_int, C.c_size_t, C.POINTER(_vp)]
_lib.tpf_comm_create_local_group.argtypes = [C.c_int, C.c_size_t, C.POINTER(_vp)]
_lib.tpf_comm_ipc_handle.argtypes = [_vp, _vp]
_lib.tpf_comm_open_peers.argtypes = [_vp, _vp]
_lib.tpf_comm_destroy.argtypes = [_vp]
_lib.tpf_comm_sync.argtypes = [_vp, _vp]
_lib.tpf_comm_set_timeout_ns.argtypes = [_vp, _i64]
_lib.tpf_comm_inject_fault.argtypes = [_vp, C.c_int]
_lib.tpf_comm_set_compute_only.argtypes = [_vp, C.c_int]
_lib.tpf_comm_set_trace.argtypes = [_vp, _vp, _i64]
_lib.tpf_ag_gemm.argtypes = [_vp, _vp, _vp, _vp] + [_i64] * 4 + [C.c_int] * 3 + [_vp]
_lib.tpf_gemm_rs.argtypes = [_vp, _vp, _vp, _vp] + [_i64] * 4 + [C.c_int] * 4 + [_vp]
_lib.tpf_gemm.argtypes = [_vp, _vp, _vp] + [_i64] * 3 + [C.c_int, _vp]
_lib.tpf_dp_grad_rs.argtypes = [_vp, _vp, _vp, _vp] + [_i64] * 3 + [C.c_int] * 4 + [_vp]
_lib.tpf_dp_param_ag_gemm.argtypes = [_vp, _vp, _vp, _vp] + [_i64] * 3 + [C.c_int, _vp]
_lib.tpf_attention_a2a.argtypes = [_vp] * 5 + [_i64] * 4 + [C.c_int, _vp]
_lib.tpf_query_split_attention.argtypes = [_vp] * 6 + [_i64] * 5 + [C.c_int] * 4 + [_vp]
_lib.tpf_ulysses_a2a.argtypes = [_vp] * 7 + [_i64] * 4 + [_vp]
_lib.tpf_ulysses_attention.argtypes = [_vp] * 5 + [_i64] * 4 + [C.c_int, _vp]
_lib.tpf_sym_bytes_ulysses.argtypes = [C.c_int] + [_i64] * 4
_lib.tpf_sym_bytes_ulysses.restype = _i64
_lib.tpf_sym_bytes_dp_ag.argtypes = [C.c_int, _i64, _i64]
_lib.tpf_sym_bytes_dp_ag.restype = _i64
_lib.tpf_swiglu.argtypes = [_vp, _vp, _i64, _i64, _vp]
_lib.tpf_sym_bytes_ag.argtypes = [C.c_int] + [_i64] * 4 + [C.c_int]
_lib.tpf_sym_bytes_ag.restype = _i64
_lib.tpf_sym_bytes_rs.argtypes = [C.c_int] + [_i64] * 4 + [C.c_int, C.c_int]
_lib.tpf_sym_bytes_rs.restype = _i64

EXPORTED_SYMBOLS = (
    "tpf_version",
    "tpf_last_error",
    "tpf_device_sms",
    "tpf_ring_indices",
    "tpf_schedule_build",
    "tpf_schedule_check",
    "tpf_comm_create",
    "tpf_comm_create_virtual",
    "tpf_comm_ipc_handle",
    "tpf_comm_open_peers",
    "tpf_comm_create_local_group",
    "tpf_comm_destroy",
    "tpf_comm_rank",
    "tpf_comm_world",
    "tpf_comm_sync",
    "tpf_comm_set_timeout_ns",
    "tpf_comm_inject_fault",
    "tpf_comm_set_compute_only",
    "tpf_comm_set_trace",
    "tpf_ag_gemm",
    "tpf_gemm_rs",
    "tpf_dp_grad_rs",
    "tpf_attention_a2a",
    "tpf_query_split_attention",
    "tpf_ulysses_a2a",
    "tpf_ulysses_attention",
    "tpf_sym_bytes_ulysses",
    "tpf_dp_param_ag_gemm",
    "tpf_sym_bytes_dp_ag",
    "tpf_gemm",
    "tpf_swiglu",
    "tpf_sym_bytes_ag",
    "tpf_sym_bytes_rs",
)


def lib() -> C.CDLL:
    return _lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = _lib.tpf_last_error().decode()
    exc = {E_INVALID: ValueError, E_SHAPE: ShapeError, E_LOGIC: LogicError, E_CUDA: TpfCudaError,
           E_PEER: GroupError, E_CAPACITY: CapacityError}.get(rc, RuntimeError)
    raise exc(msg)


# ------------------------------------------------------------------ schedules
def ring_indices_ag(r: int, i: int, n: int):
    """RingIndices ring_indices_ag(r, i, n) (collectives.cpp:47-50)."""
    out = (C.c_int32 * 3)()
    _check(_lib.tpf_ring_indices(0, r, i, n, out))
    return tuple(out)


def ring_indices_rs(r: int, i: int, n: int):
    """RingIndices ring_indices_rs(r, i, n) (collectives.cpp:52-55)."""
    out = (C.c_int32 * 3)()
    _check(_lib.tpf_ring_indices(1, r, i, n, out))
    return tuple(out)


def build_schedule(kind: int, n: int):
    """Schedule build_schedule(kind, n) -> steps[rank][iteration] = (send, recv, slice)."""
    buf = (C.c_int32 * max(1, n * n * 3))()
    _check(_lib.tpf_schedule_build(kind, n, buf))
    if n == 1:
        return [[]]
    return [[tuple(buf[(r * n + i) * 3:(r * n + i) * 3 + 3]) for i in range(n)] for r in range(n)]


def check_schedule(kind: int, steps) -> None:
    """void check_schedule(const Schedule&): raises LogicError on violation."""
    n = len(steps)
    flat = [v for row in steps for st in row for v in st]
    buf = (C.c_int32 * max(1, len(flat)))(*flat)
    _check(_lib.tpf_schedule_check(kind, n, buf))


# --------------------------------------------------------------- communicator
def _stream_ptr(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class Communicator:
    """RankEndpoint analogue (fabric.hpp:114-147) over a CUDA-IPC symmetric heap.

    * ``Communicator.local_group(world, ...)`` — all ranks hosted on the current
      GPU, every fused call runs the whole group in one persistent launch.
    * ``Communicator.from_process_group(pg, ...)`` — one process per GPU; IPC
      handles exchanged with torch.distributed (plumbing only).
    """

    def __init__(self, handle: int, rank: int, world: int, local_group: bool):
        self._h = C.c_void_p(handle)
        self.rank, self.world, self.is_local_group = rank, world, local_group

    @classmethod
    def local_group(cls, world: int, sym_bytes_per_rank: int) -> "Communicator":
        h = C.c_void_p()
        _check(_lib.tpf_comm_create_local_group(world, sym_bytes_per_rank, C.byref(h)))
        return cls(h.value, 0, world, True)

    @classmethod
    def virtual_group(cls, world: int, sym_bytes: int) -> "Communicator":
        """Performance-only: rank 0 of a `world`-rank group with virtual peers. The peers alias
        this rank's own heap (a self-ring): each send fills the slot this rank reads one step
        later, so the ring's step-to-step waits are real (zero link latency). Per-rank
        tensors, full-GPU scale; results are meaningless. See tpf_comm_create_virtual."""
        h = C.c_void_p()
        _check(_lib.tpf_comm_create_virtual(world, sym_bytes, C.byref(h)))
        return cls(h.value, 0, world, False)

    @classmethod
    def create(cls, rank: int, world: int, sym_bytes: int) -> "Communicator":
        h = C.c_void_p()
        _check(_lib.tpf_comm_create(rank, world, sym_bytes, C.byref(h)))
        return cls(h.value, rank, world, False)

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(IPC_HANDLE_BYTES)
        _check(_lib.tpf_comm_ipc_handle(self._h, buf))
        return buf.raw

    def open_peers(self, handles: Sequence[bytes]) -> None:
        blob = b"".join(handles)
        assert len(blob) == IPC_HANDLE_BYTES * self.world
        _check(_lib.tpf_comm_open_peers(self._h, C.c_char_p(blob)))

    @classmethod
    def from_process_group(cls, sym_bytes: int, group=None) -> "Communicator":
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        from .dist import exchange_ipc_handles
        comm = cls.create(rank, world, sym_bytes)
        if world > 1:
            comm.open_peers(exchange_ipc_handles(comm.ipc_handle(), group))
            dist.barrier(group)
        return comm

    def set_timeout_ms(self, ms: float) -> None:
        _check(_lib.tpf_comm_set_timeout_ns(self._h, int(ms * 1e6)))

    def inject_fault(self, rank: int) -> None:
        """Test hook: `rank` stops publishing flags (-1 clears)."""
        _check(_lib.tpf_comm_inject_fault(self._h, rank))

    def set_compute_only(self, on: bool) -> None:
        """Measurement hook: same kernels, no flag waits / wire traffic (exposed-comm baseline)."""
        _check(_lib.tpf_comm_set_compute_only(self._h, int(bool(on))))

    def set_trace(self, buf) -> None:
        """Attach a zeroed device int64 tensor of (cap+1)*4 words as the timeline trace (None: off)."""
        if buf is None:
            _check(_lib.tpf_comm_set_trace(self._h, None, 0))
        else:
            _check(_lib.tpf_comm_set_trace(self._h, buf.data_ptr(), buf.numel() // 4 - 1))

    def sync(self, stream=None) -> None:
        """Synchronise the stream and raise GroupError if a peer wait timed out."""
        _check(_lib.tpf_comm_sync(self._h, _stream_ptr(stream)))

    def close(self) -> None:
        if self._h:
            _lib.tpf_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ fused ops
    def ag_gemm(self, x, w, out, m: int = 1, act: int = ACT_NONE, stream=None) -> None:
        """column_parallel_forward / fuse_all_gather (layers.cpp:120-127).

        Per rank x: (B, S/T, K) bf16, w: (K, N_local) bf16, out: (B, S, N_local).
        A local group takes rank-stacked tensors (T, ...)."""
        lead = 1 if self.is_local_group else 0
        B, sl, K = x.shape[lead:]
        N = w.shape[-1]
        _check(_lib.tpf_ag_gemm(self._h, x.data_ptr(), w.data_ptr(), out.data_ptr(), B,
                                sl * self.world, K, N, m, act, _dtype_code(out), _stream_ptr(stream)))

    def gemm_rs(self, x, w, out, kind: int = RING, m: int = 1, wire: int = F32, stream=None) -> None:
        """row_parallel_forward / fuse_reduce_scatter (layers.cpp:129-138).

        Per rank x: (B, S, K_local) bf16, w: (K_local, N) bf16, out: (B, S/T, N)."""
        lead = 1 if self.is_local_group else 0
        B, S, K = x.shape[lead:]
        N = w.shape[-1]
        _check(_lib.tpf_gemm_rs(self._h, x.data_ptr(), w.data_ptr(), out.data_ptr(), B, S, K, N,
                                kind, m, wire, _dtype_code(out), _stream_ptr(stream)))

    def dp_grad_rs(self, X, dY, dW, kind: int = RING, m: int = 1, wire: int = F32, stream=None) -> None:
        """DP gradient reduce-scatter fused into the weight-gradient GEMM (cfg 4):
        dW_r = rows [r*K/T, (r+1)*K/T) of sum_q X_q^T dY_q. Per rank X: (M_local, K), dY: (M_local, N),
        dW: (K/T, N); a local group takes rank-stacked tensors."""
        M_local, K = X.shape[-2:]
        N = dY.shape[-1]
        _check(_lib.tpf_dp_grad_rs(self._h, X.data_ptr(), dY.data_ptr(), dW.data_ptr(), M_local, K, N, kind, m,
                                   wire, _dtype_code(dW), _stream_ptr(stream)))

    def dp_param_ag_gemm(self, x, w_rows, out, stream=None) -> None:
        """DP parameter all-gather fused into the forward GEMM (cfg 4, a19): out = x . W^T where
        W (N x K) is row-sharded over the ranks (PyTorch Linear layout). Per rank x: (M_local, K),
        w_rows: (N/T, K), out: (M_local, N); a local group takes rank-stacked tensors."""
        M_local, K = x.shape[-2:]
        N_local = w_rows.shape[-2]
        _check(_lib.tpf_dp_param_ag_gemm(self._h, x.data_ptr(), w_rows.data_ptr(), out.data_ptr(), M_local, K,
                                         N_local, _dtype_code(out), _stream_ptr(stream)))

    def attention_a2a(self, q, k, v, out, batch: int, heads: int, scale: bool = True, stream=None) -> None:
        """fuse_all_to_all_attention (Alg. 5, layers.cpp:174-218; BASELINE cfg 5).
        Per rank q/k/v: (batch*heads, S, Dh) bf16; out: (batch, S/T, T*heads*Dh) bf16.
        A local group takes rank-stacked tensors."""
        S, Dh = q.shape[-2:]
        _check(_lib.tpf_attention_a2a(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), batch, heads,
                                      S, Dh, int(bool(scale)), _stream_ptr(stream)))

    def query_split_attention(self, q, k, v, w_o, out, batch: int, heads: int, kind: int = RING,
                               wire: int = F32, scale: bool = True, stream=None) -> None:
        """query_split_attention (Alg. 4, layers.cpp:149-172). Per rank q/k/v: (batch*heads, S, 128)
        bf16, w_o: (heads*128, D) bf16 (row shard), out: (batch, S/T, D). Local groups: rank-stacked."""
        S, Dh = q.shape[-2:]
        D = w_o.shape[-1]
        _check(_lib.tpf_query_split_attention(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), w_o.data_ptr(),
                                              out.data_ptr(), batch, heads, S, Dh, D, kind, wire, _dtype_code(out),
                                              int(bool(scale)), _stream_ptr(stream)))

    def ulysses_a2a(self, q, k, v, q_out, k_out, v_out, batch: int, heads: int, stream=None) -> None:
        """Ulysses first all-to-all (ref_all_to_all of layers_test.cpp:347-397):
        per rank q/k/v (batch*heads, S/T, Dh) bf16 with every head -> (batch*heads/T, S, Dh), this
        rank's head group over the whole sequence. Local groups: rank-stacked."""
        sl, Dh = q.shape[-2:]
        _check(_lib.tpf_ulysses_a2a(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), q_out.data_ptr(),
                                    k_out.data_ptr(), v_out.data_ptr(), batch, heads, sl * self.world, Dh,
                                    _stream_ptr(stream)))

    def ulysses_attention(self, q, k, v, out, batch: int, heads: int, scale: bool = True, stream=None) -> None:
        """The whole UP attention (Alg. 5 with its first all-to-all): sequence-sharded q/k/v
        (batch*heads, S/T, 128) per rank -> out (batch, S/T, heads*128), with both all-to-alls fused
        (peer-store inbox + fused flash attention pushing O tiles to the slice owner)."""
        sl, Dh = q.shape[-2:]
        _check(_lib.tpf_ulysses_attention(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), batch,
                                          heads, sl * self.world, Dh, int(bool(scale)), _stream_ptr(stream)))

def interleave_gate_up(gate, up, tile: int = 256):
    """Tile-interleaved gate||up shard for the fused SwiGLU epilogue (ACT_SWIGLU):
    every 256-column tile holds 128 gate columns followed by the matching 128 up
    columns. gate, up: (K, F) with F % 128 == 0 -> (K, 2F)."""
    import torch
    K, F = gate.shape
    half = tile // 2
    assert up.shape == gate.shape and F % half == 0
    return torch.stack([gate.reshape(K, F // half, half), up.reshape(K, F // half, half)],
                       dim=2).reshape(K, 2 * F)


def sym_bytes_ulysses(world, batch, heads, S, Dh=128) -> int:
    """Symmetric heap bytes per rank for ulysses_attention / ulysses_a2a / attention_a2a."""
    n = int(_lib.tpf_sym_bytes_ulysses(world, batch, heads, S, Dh))
    if n < 0:
        raise ValueError(f"sym_bytes_ulysses: S={S} / heads={heads} not divisible by world={world}")
    return n


def sym_bytes_dp_ag(world, K, N_local) -> int:
    return int(_lib.tpf_sym_bytes_dp_ag(world, K, N_local))


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise ShapeError(f"unsupported output dtype {t.dtype}")


def gemm(a, b, out, stream=None) -> None:
    """T == 1 degenerate case: out = a @ b on the tcgen05 kernel."""
    M, K = a.shape
    N = b.shape[1]
    _check(_lib.tpf_gemm(a.data_ptr(), b.data_ptr(), out.data_ptr(), M, K, N, _dtype_code(out),
                         _stream_ptr(stream)))


def swiglu(gu, out, stream=None) -> None:
    rows = gu.numel() // gu.shape[-1]
    F = gu.shape[-1] // 2
    _check(_lib.tpf_swiglu(gu.data_ptr(), out.data_ptr(), rows, F, _stream_ptr(stream)))


def sym_bytes_ag(world, B, S, K, N_local, m=1) -> int:
    return int(_lib.tpf_sym_bytes_ag(world, B, S, K, N_local, m))


def sym_bytes_rs(world, B, S, K_local, N, m=1, wire=F32) -> int:
    return int(_lib.tpf_sym_bytes_rs(world, B, S, K_local, N, m, wire))
