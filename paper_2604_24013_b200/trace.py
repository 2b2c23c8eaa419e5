"""Device timeline trace of the fused kernels (tpf_comm_set_trace) and the
measured analogue of the reference's no-tail check.

The reference checks "no communication interval ends after the rank's final
compute interval" on a *simulated* timeline (costmodel.cpp:163-176,
no_tail_check). Here the same predicate is evaluated on %globaltimer stamps
the kernel records: per rank, the last peer-flag publication (RS partial pushed
to the successor / AG image forwarded) versus the end of that rank's last
GEMM tile epilogue.
"""
from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass

TR_TILE, TR_MAINLOOP, TR_AG_PIECE, TR_WAIT_A, TR_WAIT_IN, TR_FLAG = 1, 2, 3, 4, 5, 6
TR_FLUSH, TR_EPI_LOOP, TR_PUBLISH = 7, 8, 9
KIND_NAMES = {TR_TILE: "tile", TR_MAINLOOP: "mainloop", TR_AG_PIECE: "ag_piece",
              TR_WAIT_A: "wait_wire", TR_WAIT_IN: "wait_inbox", TR_FLAG: "flag",
              TR_FLUSH: "ag_flush", TR_EPI_LOOP: "rs_epilogue_loop", TR_PUBLISH: "rs_publish"}


@dataclass
class Rec:
    kind: int
    rank: int
    block: int
    step: int
    index: int
    t0: int
    t1: int


def alloc(capacity: int, device="cuda"):
    import torch
    return torch.zeros((capacity + 1) * 4, dtype=torch.int64, device=device)


def decode(buf) -> list[Rec]:
    words = buf.cpu().tolist()
    n = min(int(words[0]), len(words) // 4 - 1)
    out = []
    for k in range(1, n + 1):
        h, idx, t0, t1 = words[4 * k: 4 * k + 4]
        h &= (1 << 64) - 1
        out.append(Rec(h & 0xFF, (h >> 8) & 0xFF, (h >> 16) & 0xFFFF, (h >> 32) & 0xFFFFFFFF, idx, t0, t1))
    return out


def summarize(recs: list[Rec]) -> dict:
    """Per-rank step spans, wait totals and the measured tail (ns)."""
    if not recs:
        return {}
    t_base = min(r.t0 for r in recs if r.t0 > 0)
    per_rank = defaultdict(lambda: defaultdict(list))
    for r in recs:
        per_rank[r.rank][r.kind].append(r)
    out = {}
    for rank, kinds in sorted(per_rank.items()):
        tiles = kinds.get(TR_TILE, [])
        # transfers: RS flags published (by the epilogue or the publisher warp), AG images forwarded
        comm = kinds.get(TR_FLAG, []) + kinds.get(TR_PUBLISH, []) + kinds.get(TR_AG_PIECE, [])
        steps = defaultdict(lambda: [None, None])
        for r in kinds.get(TR_MAINLOOP, []):
            s = steps[r.step]
            s[0] = r.t0 if s[0] is None else min(s[0], r.t0)
        for r in tiles:
            s = steps[r.step]
            s[1] = r.t1 if s[1] is None else max(s[1], r.t1)
        last_compute = max((r.t1 for r in tiles), default=0)
        last_comm = max((r.t1 for r in comm), default=0)
        out[rank] = {
            "steps_us": {st: [round((a - t_base) / 1e3, 1) if a else None, round((b - t_base) / 1e3, 1) if b else None]
                         for st, (a, b) in sorted(steps.items())},
            "wait_wire_us": round(sum(r.t1 - r.t0 for r in kinds.get(TR_WAIT_A, [])) / 1e3, 1),
            "wait_inbox_us": round(sum(r.t1 - r.t0 for r in kinds.get(TR_WAIT_IN, [])) / 1e3, 1),
            "last_compute_us": round((last_compute - t_base) / 1e3, 1),
            "last_comm_us": round((last_comm - t_base) / 1e3, 1) if last_comm else None,
            "tail_us": round(max(0, last_comm - last_compute) / 1e3, 2) if last_comm else 0.0,
        }
    return out


def no_tail(summary: dict) -> bool:
    """Measured no_tail_check: no rank publishes a transfer after its last tile."""
    return all(v["tail_us"] == 0.0 for v in summary.values())
