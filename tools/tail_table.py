"""Measured no-tail check (acceptance C4, costmodel.cpp:163-176) for every op x schedule x T,
in the local group (all ranks, one launch), the split group (per-rank launch path) and the
per-GPU virtual group (full cfg2 per-rank shapes). Per case: the worst rank's tail (last flag
publication after its last tile end, us; 0 = no tail) and the margin (last tile end minus last
publication, us).   python tools/tail_table.py > profiles/r02_tail_table.json"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf
from paper_2604_24013_b200 import trace

DEV = torch.device("cuda:0")


def summarize(bufs):
    out = {}
    for b in bufs:
        out.update(trace.summarize(trace.decode(b)))
    tails = [v["tail_us"] for v in out.values()]
    margins = [v["last_compute_us"] - (v["last_comm_us"] or 0.0) for v in out.values()]
    return {"ranks": len(out), "max_tail_us": max(tails), "min_margin_us": round(min(margins), 2),
            "no_tail": all(t == 0.0 for t in tails)}


def kinds(T):
    return [tpf.RING, tpf.CIRCULAR] + ([tpf.PAIRWISE] if T % 2 == 0 else [])


def run(comms, calls, lead):
    for _ in range(2):
        calls()
    for c in comms:
        c.sync()
    bufs = [trace.alloc(400000) for _ in comms]
    for c, b in zip(comms, bufs):
        c.set_trace(b)
    calls()
    for c in comms:
        c.sync()
        c.set_trace(None)
    return summarize(bufs)


res = {}
S, K, N = 2048, 1024, 2048
for T in (2, 4, 8):
    g = torch.Generator(device=DEV).manual_seed(T)
    xa = torch.randn((T, 1, S // T, K), device=DEV, generator=g).to(torch.bfloat16)
    wa = (torch.randn((T, K, N // T), device=DEV, generator=g) / 32).to(torch.bfloat16)
    oa = torch.empty((T, 1, S, N // T), device=DEV, dtype=torch.bfloat16)
    xr = torch.randn((T, 1, S, K // T), device=DEV, generator=g).to(torch.bfloat16)
    wr = (torch.randn((T, K // T, N), device=DEV, generator=g) / 32).to(torch.bfloat16)
    orr = torch.empty((T, 1, S // T, N), device=DEV, dtype=torch.bfloat16)
    need = max(tpf.sym_bytes_ag(T, 1, S, K, N // T), tpf.sym_bytes_rs(T, 1, S, K // T, N))
    lg = tpf.Communicator.local_group(T, need)
    res[f"local T{T} ag"] = run([lg], lambda: lg.ag_gemm(xa, wa, oa), True)
    for k in kinds(T):
        res[f"local T{T} rs {tpf.KIND_NAMES[k]}"] = run([lg], lambda: lg.gemm_rs(xr, wr, orr, kind=k), True)
    lg.close()
    sg = tpf.Communicator.split_group(T, need)
    res[f"split T{T} ag"] = run(sg, lambda: [sg[r].ag_gemm(xa[r], wa[r], oa[r]) for r in range(T)], False)
    for k in kinds(T):
        res[f"split T{T} rs {tpf.KIND_NAMES[k]}"] = run(
            sg, lambda: [sg[r].gemm_rs(xr[r], wr[r], orr[r], kind=k) for r in range(T)], False)
    for c in sg:
        c.close()
    # per GPU, full cfg2 per-rank shapes
    Sv, D, F = 8192, 4096, 14336
    x = torch.randn((1, Sv // T, D), device=DEV, generator=g).to(torch.bfloat16)
    w = (torch.randn((D, 2 * F // T), device=DEV, generator=g) / 64).to(torch.bfloat16)
    act = torch.empty((1, Sv, F // T), device=DEV, dtype=torch.bfloat16)
    wd = (torch.randn((F // T, D), device=DEV, generator=g) / 64).to(torch.bfloat16)
    y = torch.empty((1, Sv // T, D), device=DEV, dtype=torch.bfloat16)
    vg = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, Sv, D, 2 * F // T),
                                               tpf.sym_bytes_rs(T, 1, Sv, F // T, D, 1, tpf.BF16)))
    res[f"virtual T{T} cfg2 ag+swiglu"] = run([vg], lambda: vg.ag_gemm(x, w, act, act=tpf.ACT_SWIGLU), False)
    for k in kinds(T):
        res[f"virtual T{T} cfg2 rs {tpf.KIND_NAMES[k]}"] = run(
            [vg], lambda: vg.gemm_rs(act, wd, y, kind=k, wire=tpf.BF16), False)
    vg.close()
    print(json.dumps({k: v for k, v in res.items() if f"T{T} " in k}), file=sys.stderr, flush=True)
print(json.dumps({"what": "measured no_tail_check per case (worst rank): tail = last flag publication after "
                          "the rank's last tile end; margin = last tile end - last publication (us)",
                  "cases": res, "all_no_tail": all(v["no_tail"] for v in res.values())}, indent=1))
