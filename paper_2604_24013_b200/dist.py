"""Multi-process host plumbing for one-rank-per-GPU groups (torch.distributed is
used only as the bootstrap / control channel; data moves in-kernel over NVLink).

* exchange_ipc_handles  — the out-of-band IPC-handle exchange tpf_comm_open_peers needs
                          (the RankGroup construction of the reference, fabric.hpp:151-174).
* sequence / feature / row / column shards — exactly the rank -> slice maps of the
  reference (split_seq tensor.cpp:145-165, ShardedLinear::split_rows/split_columns
  layers.cpp:10-48), so every rank hands the kernel the operand the reference would.
* max_over_ranks        — multi-GPU timings are reported as the max over ranks.
* simulate_ring_reduce_scatter — host replay of the data movement the fused GEMM-RS
  kernel performs, driven by the same schedule table and slot indexing (message of
  step i lands in the receiver's slot pass*(T-1)+i), over torch.distributed P2P. Used by
  the CPU (gloo) tests to check the multi-rank protocol end to end.
"""
from __future__ import annotations

from typing import List, Sequence


def exchange_ipc_handles(handle: bytes, group=None) -> List[bytes]:
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out: List[bytes] = [b""] * world
    dist.all_gather_object(out, handle, group=group)
    for r, h in enumerate(out):
        if not isinstance(h, (bytes, bytearray)) or len(h) != len(handle):
            raise RuntimeError(f"rank {r} sent a malformed IPC handle")
    return [bytes(h) for h in out]


def seq_shard(x, world: int, rank: int):
    """split_seq(x, world)[rank] for x (B, S, D): rows [rank*S/T, (rank+1)*S/T) of every batch row."""
    B, S, D = x.shape
    if S % world:
        raise ValueError(f"split_seq: sequence length {S} is not divisible by {world}")
    sl = S // world
    return x[:, rank * sl:(rank + 1) * sl].contiguous()


def feature_shard(x, world: int, rank: int):
    """Columns [rank*D/T, (rank+1)*D/T) of x (B, S, D) (row-parallel input)."""
    D = x.shape[-1]
    if D % world:
        raise ValueError(f"feature width {D} is not divisible by {world}")
    dl = D // world
    return x[..., rank * dl:(rank + 1) * dl].contiguous()


def row_shard(w, world: int, rank: int):
    """ShardedLinear::split_rows(w, world).shard(rank)."""
    K = w.shape[0]
    if K % world:
        raise ValueError(f"split_rows: {K} rows cannot be split across {world} ranks")
    kl = K // world
    return w[rank * kl:(rank + 1) * kl].contiguous()


def column_shard(w, world: int, rank: int):
    """ShardedLinear::split_columns(w, world).shard(rank)."""
    N = w.shape[1]
    if N % world:
        raise ValueError(f"split_columns: {N} columns cannot be split across {world} ranks")
    nl = N // world
    return w[:, rank * nl:(rank + 1) * nl].contiguous()


def max_over_ranks(value: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return value
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def simulate_ring_reduce_scatter(partials: Sequence, steps, m: int, group=None):
    """Replay the fused GEMM-RS data movement for this rank.

    partials[c] = this rank's f(chunk c) for the T*m sequence chunks (torch tensors,
    fp64 for exactness); steps = this rank's row of the schedule table
    [(send, recv, slice)] * T. Ring / circular kinds (pipelined: partial += inbox, then
    forward). Returns this rank's (pass-concatenated) output.
    """
    import torch
    import torch.distributed as dist
    T = len(steps)
    outs = []
    for p in range(m):
        inbox = None
        for i, (send, recv, sl) in enumerate(steps):
            part = partials[sl * m + p].clone()
            if inbox is not None:
                part = part + inbox  # rs_pipelined: partial += inbox (collectives.cpp:303)
            if i < T - 1:
                buf = torch.empty_like(part)
                ops = [dist.P2POp(dist.isend, part, send, group=group),
                       dist.P2POp(dist.irecv, buf, recv, group=group)]
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
                inbox = buf
            else:
                outs.append(part)
    return torch.cat(outs, dim=-2)
