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
    """tpfuse::GroupError (fabric.hpp:22-31): names the first failing rank. Here a rank fails
    when it stops delivering its peer flags; the ranks blocked on it (directly or through a
    chain of waits) time out and follow the blame chain back to it."""

    def __init__(self, msg: str, rank: int = -1):
        super().__init__(msg)
        if rank < 0 and msg.startswith("rank "):
            try:
                rank = int(msg.split()[1])
            except ValueError:
                rank = -1
        self._rank = rank

    def failing_rank(self) -> int:
        return self._rank


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
_lib.tpf_comm_create_split_group.argtypes = [C.c_int, C.c_size_t, C.POINTER(_vp)]
_lib.tpf_comm_failing_rank.argtypes = [_vp]
_lib.tpf_comm_ipc_handle.argtypes = [_vp, _vp]
_lib.tpf_comm_open_peers.argtypes = [_vp, _vp]
_lib.tpf_comm_destroy.argtypes = [_vp]
_lib.tpf_comm_device.argtypes = [_vp]
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
    "tpf_comm_create_split_group",
    "tpf_comm_failing_rank",
    "tpf_comm_destroy",
    "tpf_comm_rank",
    "tpf_comm_world",
    "tpf_comm_device",
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


# ------------------------------------------------------------ argument checks
# The C ABI takes raw pointers, so every wrapper checks dtype, layout, device and the exact
# shape of each tensor first and raises ShapeError naming both shapes, as the reference's
# matmul / accumulate do (tensor.cpp:68-85, 215-221; tensor.hpp:13-16).
def _require(t, name: str, shape, dtypes=("bf16",), device=None) -> None:
    import torch
    names = {"bf16": torch.bfloat16, "f32": torch.float32}
    if not isinstance(t, torch.Tensor):
        raise ShapeError(f"{name}: expected a torch.Tensor, got {type(t).__name__}")
    if tuple(t.shape) != tuple(shape):
        raise ShapeError(f"{name}: shape {tuple(t.shape)} does not match the expected {tuple(shape)}")
    if t.dtype not in [names[d] for d in dtypes]:
        raise ShapeError(f"{name}: dtype {t.dtype} not supported (expected {' or '.join(dtypes)})")
    if not t.is_contiguous():
        raise ShapeError(f"{name}: tensor must be contiguous (row-major), got strides {tuple(t.stride())}")
    if device is not None and t.device != device:
        raise ShapeError(f"{name}: tensor is on {t.device}, the communicator on {device}")
    elif device is None and t.device.type != "cuda":
        raise ShapeError(f"{name}: tensor must be on a CUDA device, got {t.device}")


OUT_DTYPES = ("bf16", "f32")


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

    def __init__(self, handle: int, rank: int, world: int, local_group: bool, device=None):
        self._h = C.c_void_p(handle)
        self.rank, self.world, self.is_local_group = rank, world, local_group
        if device is None:
            import torch
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        # The library links its own (static) CUDA runtime. It must see the device torch made
        # current, or its kernels would run on another GPU than the tensors they are given.
        lib_dev = _lib.tpf_comm_device(self._h)
        if lib_dev != device.index:
            _lib.tpf_comm_destroy(self._h)
            raise TpfCudaError(f"communicator created on device {lib_dev}, but the tensors' device is "
                               f"cuda:{device.index} (call torch.cuda.set_device first)")

    def _lead(self):
        # local groups take rank-stacked tensors: a leading dim of `world`
        return (self.world,) if self.is_local_group else ()

    def _dims(self, t, name: str, nd: int):
        import torch
        if not isinstance(t, torch.Tensor):
            raise ShapeError(f"{name}: expected a torch.Tensor, got {type(t).__name__}")
        lead = self._lead()
        if t.dim() != len(lead) + nd or tuple(t.shape[:len(lead)]) != lead:
            want = "(" + ", ".join([str(w) for w in lead] + ["*"] * nd) + ")"
            raise ShapeError(f"{name}: shape {tuple(t.shape)} does not match {want}")
        return tuple(t.shape[len(lead):])

    @classmethod
    def local_group(cls, world: int, sym_bytes_per_rank: int) -> "Communicator":
        h = C.c_void_p()
        _check(_lib.tpf_comm_create_local_group(world, sym_bytes_per_rank, C.byref(h)))
        return cls(h.value, 0, world, True)

    @classmethod
    def split_group(cls, world: int, sym_bytes: int) -> list:
        """`world` per-rank communicators on the current GPU (tpf_comm_create_split_group):
        each is a one-process-per-GPU communicator (its own heap, device epoch and error
        record; per-rank tensors, no stacking) whose peers are the others' heaps. A fused GEMM
        call on every rank (any order, same stream) runs as one launch once the last rank has
        made it. Proves the per-rank protocol with real waits on one GPU."""
        hs = (_vp * world)()
        _check(_lib.tpf_comm_create_split_group(world, sym_bytes, hs))
        return [cls(hs[r], r, world, False) for r in range(world)]

    @classmethod
    def virtual_group(cls, world: int, sym_bytes: int) -> "Communicator":
        """Measurement tool: rank 0 of a `world`-rank group with virtual peers. The peers alias
        this rank's own heap (a self-ring): each send fills the slot this rank reads one step
        later, so the ring's step-to-step waits are real (zero link latency). Per-rank
        tensors, full-GPU scale. Results are well defined but not a real group's (the AG
        gathers the own slice every step, the GEMM-RS sums every row slice's GEMM;
        tests/test_gpu_virtual.py). See tpf_comm_create_virtual."""
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
        """Synchronise the stream and raise GroupError (naming the failing rank, not the
        rank that timed out) if a peer wait gave up."""
        rc = _lib.tpf_comm_sync(self._h, _stream_ptr(stream))
        if rc == E_PEER:
            raise GroupError(_lib.tpf_last_error().decode(), int(_lib.tpf_comm_failing_rank(self._h)))
        _check(rc)

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
        B, sl, K = self._dims(x, "ag_gemm x", 3)
        L, dev = self._lead(), self.device
        N = self._dims(w, "ag_gemm w", 2)[1]
        _require(x, "ag_gemm x", L + (B, sl, K), device=dev)
        _require(w, "ag_gemm w", L + (K, N), device=dev)
        if m >= 1 and (self.world == 1 or sl % m == 0):  # else the library raises the reference's error
            _require(out, "ag_gemm out", L + (B, sl * self.world, N // 2 if act == ACT_SWIGLU else N), OUT_DTYPES,
                     dev)
        _check(_lib.tpf_ag_gemm(self._h, x.data_ptr(), w.data_ptr(), out.data_ptr(), B,
                                sl * self.world, K, N, m, act, _dtype_code(out), _stream_ptr(stream)))

    def gemm_rs(self, x, w, out, kind: int = RING, m: int = 1, wire: int = F32, stream=None) -> None:
        """row_parallel_forward / fuse_reduce_scatter (layers.cpp:129-138).

        Per rank x: (B, S, K_local) bf16, w: (K_local, N) bf16, out: (B, S/T, N)."""
        B, S, K = self._dims(x, "gemm_rs x", 3)
        L, dev = self._lead(), self.device
        N = self._dims(w, "gemm_rs w", 2)[1]
        _require(x, "gemm_rs x", L + (B, S, K), device=dev)
        _require(w, "gemm_rs w", L + (K, N), device=dev)
        if m >= 1 and S % (self.world * m) == 0:  # else the library raises the reference's error
            _require(out, "gemm_rs out", L + (B, S // self.world, N), OUT_DTYPES, dev)
        _check(_lib.tpf_gemm_rs(self._h, x.data_ptr(), w.data_ptr(), out.data_ptr(), B, S, K, N,
                                kind, m, wire, _dtype_code(out), _stream_ptr(stream)))

    def dp_grad_rs(self, X, dY, dW, kind: int = RING, m: int = 1, wire: int = F32, stream=None) -> None:
        """DP gradient reduce-scatter fused into the weight-gradient GEMM (cfg 4):
        dW_r = rows [r*K/T, (r+1)*K/T) of sum_q X_q^T dY_q. Per rank X: (M_local, K), dY: (M_local, N),
        dW: (K/T, N); a local group takes rank-stacked tensors."""
        M_local, K = self._dims(X, "dp_grad_rs X", 2)
        N = self._dims(dY, "dp_grad_rs dY", 2)[1]
        L, dev = self._lead(), self.device
        _require(X, "dp_grad_rs X", L + (M_local, K), device=dev)
        _require(dY, "dp_grad_rs dY", L + (M_local, N), device=dev)
        if K % self.world == 0:
            _require(dW, "dp_grad_rs dW", L + (K // self.world, N), OUT_DTYPES, dev)
        _check(_lib.tpf_dp_grad_rs(self._h, X.data_ptr(), dY.data_ptr(), dW.data_ptr(), M_local, K, N, kind, m,
                                   wire, _dtype_code(dW), _stream_ptr(stream)))

    def dp_param_ag_gemm(self, x, w_rows, out, stream=None) -> None:
        """DP parameter all-gather fused into the forward GEMM (cfg 4, a19): out = x . W^T where
        W (N x K) is row-sharded over the ranks (PyTorch Linear layout). Per rank x: (M_local, K),
        w_rows: (N/T, K), out: (M_local, N); a local group takes rank-stacked tensors."""
        M_local, K = self._dims(x, "dp_param_ag_gemm x", 2)
        N_local = self._dims(w_rows, "dp_param_ag_gemm w_rows", 2)[0]
        L, dev = self._lead(), self.device
        _require(x, "dp_param_ag_gemm x", L + (M_local, K), device=dev)
        _require(w_rows, "dp_param_ag_gemm w_rows", L + (N_local, K), device=dev)
        _require(out, "dp_param_ag_gemm out", L + (M_local, self.world * N_local), OUT_DTYPES, dev)
        _check(_lib.tpf_dp_param_ag_gemm(self._h, x.data_ptr(), w_rows.data_ptr(), out.data_ptr(), M_local, K,
                                         N_local, _dtype_code(out), _stream_ptr(stream)))

    def attention_a2a(self, q, k, v, out, batch: int, heads: int, scale: bool = True, stream=None) -> None:
        """fuse_all_to_all_attention (Alg. 5, layers.cpp:174-218; BASELINE cfg 5).
        Per rank q/k/v: (batch*heads, S, Dh) bf16; out: (batch, S/T, T*heads*Dh) bf16.
        A local group takes rank-stacked tensors."""
        G, S, Dh = self._dims(q, "attention_a2a q", 3)
        L, dev, T = self._lead(), self.device, self.world
        if G != batch * heads:
            raise ShapeError(f"attention_a2a q: {G} head rows != batch {batch} x heads {heads}")
        for name, t in (("q", q), ("k", k), ("v", v)):
            _require(t, f"attention_a2a {name}", L + (G, S, Dh), device=dev)
        if S % T == 0:
            _require(out, "attention_a2a out", L + (batch, S // T, T * heads * Dh), ("bf16",), dev)
        _check(_lib.tpf_attention_a2a(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), batch, heads,
                                      S, Dh, int(bool(scale)), _stream_ptr(stream)))

    def query_split_attention(self, q, k, v, w_o, out, batch: int, heads: int, kind: int = RING,
                               wire: int = F32, scale: bool = True, stream=None) -> None:
        """query_split_attention (Alg. 4, layers.cpp:149-172). Per rank q/k/v: (batch*heads, S, 128)
        bf16, w_o: (heads*128, D) bf16 (row shard), out: (batch, S/T, D). Local groups: rank-stacked."""
        G, S, Dh = self._dims(q, "query_split_attention q", 3)
        D = self._dims(w_o, "query_split_attention w_o", 2)[1]
        L, dev, T = self._lead(), self.device, self.world
        if G != batch * heads:
            raise ShapeError(f"query_split_attention q: {G} head rows != batch {batch} x heads {heads}")
        for name, t in (("q", q), ("k", k), ("v", v)):
            _require(t, f"query_split_attention {name}", L + (G, S, Dh), device=dev)
        _require(w_o, "query_split_attention w_o", L + (heads * Dh, D), device=dev)
        if S % T == 0:
            _require(out, "query_split_attention out", L + (batch, S // T, D), OUT_DTYPES, dev)
        _check(_lib.tpf_query_split_attention(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), w_o.data_ptr(),
                                              out.data_ptr(), batch, heads, S, Dh, D, kind, wire, _dtype_code(out),
                                              int(bool(scale)), _stream_ptr(stream)))

    def ulysses_a2a(self, q, k, v, q_out, k_out, v_out, batch: int, heads: int, stream=None) -> None:
        """Ulysses first all-to-all (ref_all_to_all of layers_test.cpp:347-397):
        per rank q/k/v (batch*heads, S/T, Dh) bf16 with every head -> (batch*heads/T, S, Dh), this
        rank's head group over the whole sequence. Local groups: rank-stacked."""
        G, sl, Dh = self._dims(q, "ulysses_a2a q", 3)
        L, dev, T = self._lead(), self.device, self.world
        if G != batch * heads:
            raise ShapeError(f"ulysses_a2a q: {G} head rows != batch {batch} x heads {heads}")
        for name, t in (("q", q), ("k", k), ("v", v)):
            _require(t, f"ulysses_a2a {name}", L + (G, sl, Dh), device=dev)
        if heads % T == 0:
            for name, t in (("q_out", q_out), ("k_out", k_out), ("v_out", v_out)):
                _require(t, f"ulysses_a2a {name}", L + (batch * heads // T, sl * T, Dh), ("bf16",), dev)
        _check(_lib.tpf_ulysses_a2a(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(), q_out.data_ptr(),
                                    k_out.data_ptr(), v_out.data_ptr(), batch, heads, sl * self.world, Dh,
                                    _stream_ptr(stream)))

    def ulysses_attention(self, q, k, v, out, batch: int, heads: int, scale: bool = True, stream=None) -> None:
        """The whole UP attention (Alg. 5 with its first all-to-all): sequence-sharded q/k/v
        (batch*heads, S/T, 128) per rank -> out (batch, S/T, heads*128), with both all-to-alls fused
        (peer-store inbox + fused flash attention pushing O tiles to the slice owner)."""
        G, sl, Dh = self._dims(q, "ulysses_attention q", 3)
        L, dev = self._lead(), self.device
        if G != batch * heads:
            raise ShapeError(f"ulysses_attention q: {G} head rows != batch {batch} x heads {heads}")
        for name, t in (("q", q), ("k", k), ("v", v)):
            _require(t, f"ulysses_attention {name}", L + (G, sl, Dh), device=dev)
        _require(out, "ulysses_attention out", L + (batch, sl, heads * Dh), ("bf16",), dev)
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
    if a.dim() != 2 or b.dim() != 2:
        raise ShapeError(f"gemm: operands must be 2-D, got {tuple(a.shape)} x {tuple(b.shape)}")
    M, K = a.shape
    N = b.shape[1]
    if b.shape[0] != K:  # matmul's ShapeError names both shapes (tensor.cpp:68-85)
        raise ShapeError(f"matmul: shape mismatch {tuple(a.shape)} x {tuple(b.shape)}")
    _require(a, "gemm a", (M, K))
    _require(b, "gemm b", (K, N), device=a.device)
    _require(out, "gemm out", (M, N), OUT_DTYPES, a.device)
    _check(_lib.tpf_gemm(a.data_ptr(), b.data_ptr(), out.data_ptr(), M, K, N, _dtype_code(out),
                         _stream_ptr(stream)))


def swiglu(gu, out, stream=None) -> None:
    F = gu.shape[-1] // 2
    _require(gu, "swiglu gu", tuple(gu.shape[:-1]) + (2 * F,))
    _require(out, "swiglu out", tuple(gu.shape[:-1]) + (F,), ("bf16",), gu.device)
    rows = gu.numel() // gu.shape[-1]
    _check(_lib.tpf_swiglu(gu.data_ptr(), out.data_ptr(), rows, F, _stream_ptr(stream)))


def sym_bytes_ag(world, B, S, K, N_local, m=1) -> int:
    return int(_lib.tpf_sym_bytes_ag(world, B, S, K, N_local, m))


def sym_bytes_rs(world, B, S, K_local, N, m=1, wire=F32) -> int:
    return int(_lib.tpf_sym_bytes_rs(world, B, S, K_local, N, m, wire))
