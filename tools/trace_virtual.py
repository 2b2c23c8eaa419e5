"""Dev tool: device timeline of one per-GPU fused op of a real TP group (virtual peers,
full 148-SM scale): per-tile main-loop and epilogue durations, the gap between a pair's
consecutive main loops (MMA idle, waiting for a free TMEM accumulator or for operands),
and the kernel span.  python tools/trace_virtual.py [T] [cfg2|cfg3]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf
from paper_2604_24013_b200 import trace

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
STEADY = "steady" in sys.argv[3:]
cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
S, K_ag, N_ag, K_rs, N_rs = {"cfg2": (8192, 4096, 28672, 14336, 4096),
                             "cfg3": (16384, 8192, 10240, 8192, 8192)}[cfg]
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn((1, S // T, K_ag), device=dev, generator=g).to(torch.bfloat16)
w = (torch.randn((K_ag, N_ag // T), device=dev, generator=g) / 64).to(torch.bfloat16)
y = torch.empty((1, S, N_ag // T), device=dev, dtype=torch.bfloat16)
xr = torch.randn((1, S, K_rs // T), device=dev, generator=g).to(torch.bfloat16)
wr = (torch.randn((K_rs // T, N_rs), device=dev, generator=g) / 64).to(torch.bfloat16)
yr = torch.empty((1, S // T, N_rs), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, K_ag, N_ag // T),
                                             tpf.sym_bytes_rs(T, 1, S, K_rs // T, N_rs, 1, tpf.BF16)))


def show(name, fn, compute_only=False):
    comm.set_compute_only(compute_only)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    buf = trace.alloc(400000)
    torch.cuda._sleep(2_000_000)  # keep the GPU busy while the host enqueues the traced call
    if STEADY:  # the traced call runs between back-to-back calls, as in the timed loops
        for _ in range(3):
            fn()
    comm.set_trace(buf)
    fn()
    comm.set_trace(None)
    if STEADY:
        for _ in range(3):
            fn()
    comm.sync()
    comm.set_compute_only(False)
    recs = trace.decode(buf)
    t0 = min(r.t0 for r in recs if r.t0 > 0)
    ml = [r for r in recs if r.kind == trace.TR_MAINLOOP]
    ep = [r for r in recs if r.kind == trace.TR_TILE]
    span = max(r.t1 for r in recs) - t0
    by = {}
    for r in ml:
        by.setdefault(r.block, []).append(r)
    gaps, first, last = [], [], []
    for v in by.values():
        v = sorted(v, key=lambda r: r.t0)
        first.append((v[0].t0 - t0) / 1e3)
        last.append((v[-1].t1 - t0) / 1e3)
        gaps += [(b.t0 - a.t1) / 1e3 for a, b in zip(v, v[1:])]
    mlm = sum(r.t1 - r.t0 for r in ml) / len(ml) / 1e3
    epm = sum(r.t1 - r.t0 for r in ep) / max(1, len(ep)) / 1e3
    print(f"{name}{' (compute-only)' if compute_only else ''}: span {span / 1e3:.1f} us, {len(ml)} main loops "
          f"mean {mlm:.2f} us, {len(ep)} epilogues mean {epm:.2f} us (max {max(r.t1 - r.t0 for r in ep) / 1e3:.2f}), "
          f"MMA gap between tiles mean {sum(gaps) / max(1, len(gaps)):.2f} max {max(gaps or [0]):.2f} us, "
          f"first main loop starts {min(first):.1f}-{max(first):.1f} us, last ends {min(last):.1f}-{max(last):.1f} us",
          flush=True)
    # per-pair load balance: total producer main-loop time per block, and the blocks
    # (SM placement follows blockIdx) that finish last
    busy = sorted((sum(r.t1 - r.t0 for r in v) / 1e3, b) for b, v in by.items())
    fin = sorted(((max(r.t1 for r in v) - t0) / 1e3, b) for b, v in by.items())
    print(f"    per-block main-loop busy: min {busy[0][0]:.1f} median {busy[len(busy) // 2][0]:.1f} max {busy[-1][0]:.1f} us;"
          f" slowest blocks {[b for _, b in busy[-6:]]}, last to finish {[b for _, b in fin[-6:]]}", flush=True)
    # per step: first main-loop start, last main-loop end, last epilogue end (us from t0)
    steps = {}
    tk = min(r.t0 for r in recs if r.t0 > 0)
    for r in ml:
        st = steps.setdefault(r.step, [1e18, 0, 0])
        st[1] = max(st[1], r.t1)
    for r in ep:
        steps.setdefault(r.step, [1e18, 0, 0])[2] = max(steps[r.step][2], r.t1)
    print("    steps (mainloop last end / last epilogue end, us): " +
          " ".join(f"{k}:{(v[1] - tk) / 1e3:.0f}/{(v[2] - tk) / 1e3:.0f}"
                   for k, v in sorted(steps.items())), flush=True)
    for kind in (trace.TR_EPI_LOOP, trace.TR_PUBLISH, trace.TR_FLUSH, trace.TR_WAIT_IN, trace.TR_WAIT_A):
        rr = [r for r in recs if r.kind == kind]
        if rr:
            print(f"    {trace.KIND_NAMES[kind]}: {len(rr)} records, mean {sum(r.t1 - r.t0 for r in rr) / len(rr) / 1e3:.2f} us, "
                  f"max {max(r.t1 - r.t0 for r in rr) / 1e3:.2f} us", flush=True)


show("AG", lambda: comm.ag_gemm(x, w, y))
show("AG", lambda: comm.ag_gemm(x, w, y), True)
if "pairwise" in sys.argv[3:]:
    show("RS pairwise", lambda: comm.gemm_rs(xr, wr, yr, kind=tpf.PAIRWISE, wire=tpf.BF16))
show("RS", lambda: comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=tpf.BF16))
show("RS", lambda: comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=tpf.BF16), True)
comm.close()
