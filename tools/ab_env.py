"""Dev tool: A/B environment settings on the bench workloads, alternating processes (cancels
power-cap drift). Each process prints the T = 1 Llama-3-8B MLP block TFLOP/s and the per-GPU
TP = 8 block (virtual peers: AG-GEMM + SwiGLU, then GEMM-RS) in us per op.
    python tools/ab_env.py 'TPF_PDL=0' 'TPF_PDL=1' ['TPF_PDL=2' ...] [--rounds 3]"""
import os
import statistics
import subprocess
import sys

CODE = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2604_24013_b200 as tpf
dev = torch.device("cuda:0")
S, D, F = 8192, 4096, 14336
g = torch.Generator(device=dev).manual_seed(0)
def loop(fn, n):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
x = torch.randn((1, S, D), device=dev, generator=g).to(torch.bfloat16)
wgu = (torch.randn((D, 2 * F), device=dev, generator=g) / 64).to(torch.bfloat16)
wdn = (torch.randn((F, D), device=dev, generator=g) / 120).to(torch.bfloat16)
act = torch.empty((1, S, F), device=dev, dtype=torch.bfloat16)
y = torch.empty((1, S, D), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.create(0, 1, 0)
ms = loop(lambda: (comm.ag_gemm(x, wgu, act, act=tpf.ACT_SWIGLU), comm.gemm_rs(act, wdn, y)), 60)
t1 = (2.0 * S * D * 2 * F + 2.0 * S * F * D) / (ms * 1e-3) / 1e12
T = 8
xs, ws, ys = x[:, :S // T].contiguous(), wgu[:, :2 * F // T].contiguous(), act[:, :, :F // T].contiguous()
wd, yd = wdn[:F // T].contiguous(), y[:, :S // T].contiguous()
v = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, D, 2 * F // T, 1),
                                          tpf.sym_bytes_rs(T, 1, S, F // T, D, 1, tpf.BF16)))
ag = loop(lambda: v.ag_gemm(xs, ws, ys, act=tpf.ACT_SWIGLU), 40)
rs = loop(lambda: v.gemm_rs(ys, wd, yd, kind=tpf.RING, wire=tpf.BF16), 40)
blk = loop(lambda: (v.ag_gemm(xs, ws, ys, act=tpf.ACT_SWIGLU), v.gemm_rs(ys, wd, yd, kind=tpf.RING, wire=tpf.BF16)), 40)
print(f"{t1:.1f} {1e3 * ag:.1f} {1e3 * rs:.1f} {1e3 * blk:.1f}")
'''
args = [a for a in sys.argv[1:] if not a.startswith("--")]
rounds = 3
if "--rounds" in sys.argv:
    rounds = int(sys.argv[sys.argv.index("--rounds") + 1])
    args = [a for a in args if a != str(rounds)]
res = {e: [] for e in args}
for _ in range(rounds):
    for e in args:
        env = dict(os.environ)
        for kv in e.split():
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=300)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else ""
        res[e].append([float(t) for t in line.split()] if line else None)
        if not line:
            print(e, "failed:", out.stderr[-2000:], flush=True)
print("env: T=1 block TF/s | TP8 per-GPU AG+SwiGLU us | RS us | AG+RS block us   (median over rounds)")
for e in args:
    ok = [r for r in res[e] if r]
    if ok:
        med = [statistics.median(c) for c in zip(*ok)]
        print(f"{e}: {med[0]:.0f} TF/s | {med[1]:.1f} | {med[2]:.1f} | {med[3]:.1f}   runs {[[round(v) for v in r] for r in ok]}")
