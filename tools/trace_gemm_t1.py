"""Dev tool: device timeline of one T = 1 GEMM (through a world-1 communicator) to see the
per-tile main-loop and epilogue durations. python tools/trace_gemm_t1.py M K N"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf
from paper_2604_24013_b200 import trace

M, K, N = (int(v) for v in sys.argv[1:4])
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn((1, M, K), device=dev, generator=g).to(torch.bfloat16)
w = (torch.randn((K, N), device=dev, generator=g) / 64).to(torch.bfloat16)
y = torch.empty((1, M, N), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.create(0, 1, 0)
for _ in range(3):
    comm.gemm_rs(x, w, y)
torch.cuda.synchronize()
buf = trace.alloc(200000)
comm.set_trace(buf)
comm.gemm_rs(x, w, y)
comm.sync()
comm.set_trace(None)
recs = trace.decode(buf)
t0 = min(r.t0 for r in recs if r.t0 > 0)
ml = [r for r in recs if r.kind == trace.TR_MAINLOOP]
ep = [r for r in recs if r.kind == trace.TR_TILE]
span = max(r.t1 for r in recs) - t0
print(f"records {len(recs)}  span {span / 1e3:.1f} us  mainloops {len(ml)} mean {sum(r.t1 - r.t0 for r in ml) / len(ml) / 1e3:.2f} us"
      f"  epilogues {len(ep)} mean {sum(r.t1 - r.t0 for r in ep) / max(1, len(ep)) / 1e3:.2f} us")
# per pair: first mainloop start, last epilogue end, busy mainloop time
by = {}
for r in ml:
    by.setdefault(r.index % 74, []).append(r)
starts = sorted(min(rr.t0 for rr in v) - t0 for v in by.values())
print("first mainloop start per pair (us): min %.1f max %.1f" % (starts[0] / 1e3, starts[-1] / 1e3))
gaps = []
for v in by.values():
    v = sorted(v, key=lambda r: r.t0)
    for a, b in zip(v, v[1:]):
        gaps.append((b.t0 - a.t1) / 1e3)
print("gap between consecutive main loops of a pair (us): mean %.2f max %.2f" % (sum(gaps) / len(gaps), max(gaps)))
