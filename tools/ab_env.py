"""Dev tool: the bench block (T = 1, Llama-3-8B MLP) under different environment settings,
alternating processes. python tools/ab_env.py 'TPF_GROUP_M=16' 'TPF_GROUP_M=32' [rounds]"""
import os
import subprocess
import sys

CODE = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2604_24013_b200 as tpf
dev = torch.device("cuda:0")
S, D, F = 8192, 4096, 14336
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn((1, S, D), device=dev, generator=g).to(torch.bfloat16)
wgu = (torch.randn((D, 2 * F), device=dev, generator=g) / 64).to(torch.bfloat16)
wdn = (torch.randn((F, D), device=dev, generator=g) / 120).to(torch.bfloat16)
act = torch.empty((1, S, F), device=dev, dtype=torch.bfloat16)
y = torch.empty((1, S, D), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.create(0, 1, 0)
def step():
    comm.ag_gemm(x, wgu, act, act=tpf.ACT_SWIGLU); comm.gemm_rs(act, wdn, y)
for _ in range(20): step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(100): step()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 100
print(2.0 * S * D * 2 * F / (ms * 1e-3) / 1e12 + 2.0 * S * F * D / (ms * 1e-3) / 1e12)
'''
envs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
res = {e: [] for e in envs}
for _ in range(rounds):
    for e in envs:
        env = dict(os.environ)
        for kv in e.split():
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=300)
        res[e].append(float(out.stdout.strip().splitlines()[-1]) if out.stdout.strip() else -1.0)
for e in envs:
    print(f"{e}: runs {[round(v) for v in res[e]]}")
