"""Dev tool: A/B the UP attention kernel of two library builds in one process pair,
alternating runs to cancel clock drift. python tools/ab_up.py LIB_A LIB_B [rounds]"""
import os
import subprocess
import sys

CODE = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2604_24013_b200 as tpf
dev = torch.device("cuda:0")
T, heads, S = 8, 4, int(os.environ.get("AB_S", "32768"))
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = (torch.randn((T, heads, S, 128), device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
o = torch.empty((T, 1, S // T, T * heads * 128), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.local_group(T, 2 * (S // T) * T * heads * 128 * 2 + (8 << 20))
for _ in range(2): comm.attention_a2a(q, k, v, o, 1, heads)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); comm.attention_a2a(q, k, v, o, 1, heads); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
comm.sync(); comm.close()
print(4.0 * T * heads * S * S * 128 / best / 1e9)
'''

libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
res = {l: [] for l in libs}
for _ in range(rounds):
    for l in libs:
        env = dict(os.environ, TPF_LIB_PATH=os.path.abspath(l))
        out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=300)
        res[l].append(float(out.stdout.strip().splitlines()[-1]))
for l in libs:
    print(f"{l}: best {max(res[l]):.0f} TF/s  runs {[round(x) for x in res[l]]}")
