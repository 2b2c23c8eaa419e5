"""Dev tool: device timeline of one fused call on a single-GPU local group.

    python tools/trace_fused.py ag|rs [T] [kind] [wire]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_24013_b200 as tpf
from paper_2604_24013_b200 import trace

dev = torch.device("cuda:0")
op = sys.argv[1] if len(sys.argv) > 1 else "ag"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8
kind = int(sys.argv[3]) if len(sys.argv) > 3 else tpf.RING
wire = int(sys.argv[4]) if len(sys.argv) > 4 else tpf.BF16
S, D, F = (int(os.environ.get(k, v)) for k, v in (("TR_S", "8192"), ("TR_D", "4096"), ("TR_F", "14336")))
g = torch.Generator(device=dev).manual_seed(0)
if op == "ag":
    x = torch.randn((T, 1, S // T, D), device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn((T, D, 2 * F // T), device=dev, generator=g) / 64).to(torch.bfloat16)
    out = torch.empty((T, 1, S, 2 * F // T), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ag(T, 1, S, D, 2 * F // T, 1))
    call = lambda: comm.ag_gemm(x, w, out)  # noqa: E731
else:
    x = torch.randn((T, 1, S, F // T), device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn((T, F // T, D), device=dev, generator=g) / 64).to(torch.bfloat16)
    out = torch.empty((T, 1, S // T, D), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_rs(T, 1, S, F // T, D, 1, wire))
    call = lambda: comm.gemm_rs(x, w, out, kind=kind, wire=wire)  # noqa: E731
for _ in range(3):
    call()
comm.sync()
buf = trace.alloc(400000)
comm.set_trace(buf)
call()
comm.sync()
comm.set_trace(None)
recs = trace.decode(buf)
summ = trace.summarize(recs)
print(f"{len(recs)} records")
for r in (0, T - 1):
    print(f"rank {r}:", json.dumps(summ[r]))
pieces = [rr for rr in recs if rr.kind == trace.TR_AG_PIECE and rr.rank == 0]
if pieces:
    t_base = min(rr.t0 for rr in recs if rr.t0 > 0)
    by_slot = {}
    for rr in pieces:
        b = by_slot.setdefault(rr.step, [1e30, 0, 0.0, 0])
        b[0] = min(b[0], rr.t0)
        b[1] = max(b[1], rr.t1)
        b[2] += rr.t1 - rr.t0
        b[3] += 1
    for sl, (a, b, d, n) in sorted(by_slot.items()):
        print(f"  rank0 AG slot {sl}: first src {(a - t_base) / 1e3:8.1f} us  last publish {(b - t_base) / 1e3:8.1f} us  "
              f"mean piece {d / n / 1e3:6.2f} us  n={n}")
print("no_tail:", trace.no_tail(summ))

# main-loop durations (every AG tile reads its operand the same way: forwarding is decoupled)
if op == "ag":
    ml = [(rr.t1 - rr.t0) / 1e3 for rr in recs if rr.kind == trace.TR_MAINLOOP and rr.rank == 0]
    print(f"rank0 mainloop(us): n={len(ml)} mean={sum(ml) / max(1, len(ml)):.1f}")
    ep = [(rr.t1 - rr.t0) / 1e3 for rr in recs if rr.kind == trace.TR_TILE and rr.rank == 0]
    print(f"rank0 epilogue(us): mean={sum(ep) / max(1, len(ep)):.1f} max={max(ep):.1f}")
    fl = [rr for rr in recs if rr.kind == 7 and rr.rank == 0]
    if fl:
        d = sorted((rr.t1 - rr.t0) / 1e3 for rr in fl)
        print(f"rank0 flush(us): n={len(d)} mean={sum(d) / len(d):.2f} p50={d[len(d) // 2]:.2f} max={d[-1]:.2f} "
              f"flags/flush={sum(rr.index for rr in fl) / len(fl):.1f}")
    # producer waits on wire images, by step
    wa = [rr for rr in recs if rr.kind == trace.TR_WAIT_A and rr.rank == 0]
    by = {}
    for rr in wa:
        by.setdefault(rr.step, [0, 0.0])
        by[rr.step][0] += 1
        by[rr.step][1] += (rr.t1 - rr.t0) / 1e3
    print("rank0 producer wire waits by step (count, total us):", {k: (v[0], round(v[1], 1)) for k, v in sorted(by.items())})
    # per-pair busy fraction: sum of mainloop spans / kernel span
    t_base = min(rr.t0 for rr in recs if rr.t0 > 0)
    t_end = max(rr.t1 for rr in recs)
    busy = {}
    for rr in ml:
        busy[rr.block] = busy.get(rr.block, 0) + (rr.t1 - rr.t0)
    print(f"rank0 kernel span {(t_end - t_base) / 1e3:.0f} us; mainloop busy per CTA (us): "
          f"min {min(busy.values()) / 1e3:.0f} max {max(busy.values()) / 1e3:.0f}")
