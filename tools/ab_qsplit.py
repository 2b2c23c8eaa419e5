"""Dev tool: query_split_attention sequential (attention launch, then GEMM-RS) vs concurrent
(attention and GEMM-RS co-resident, per-slice ready counters), alternating processes.
python tools/ab_qsplit.py [T] [S] [heads_per_rank] [D]"""
import os
import subprocess
import sys

CODE = r'''
import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_2604_24013_b200 as tpf
T, S, h, D = (int(v) for v in sys.argv[1:5])
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = (torch.randn((T, h, S, 128), device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
w = (torch.randn((T, h * 128, D), device=dev, generator=g) / 64).to(torch.bfloat16)
out = torch.empty((T, 1, S // T, D), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.local_group(T, tpf.sym_bytes_rs(T, 1, S, h * 128, D, 1, tpf.BF16) + (1 << 22))
fn = lambda: comm.query_split_attention(q, k, v, w, out, 1, h, wire=tpf.BF16)
for _ in range(3): fn()
torch.cuda.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
comm.sync(); comm.close()
print(statistics.median(ts))
'''
args = sys.argv[1:5] if len(sys.argv) > 4 else ["4", "8192", "8", "4096"]
res = {"0": [], "1": []}
for _ in range(3):
    for mode in ("0", "1"):
        env = dict(os.environ, TPF_QSPLIT_CONCURRENT=mode)
        out = subprocess.run([sys.executable, "-c", CODE] + args, env=env, capture_output=True, text=True, timeout=300)
        res[mode].append(float(out.stdout.strip().splitlines()[-1]) if out.stdout.strip() else -1.0)
        if not out.stdout.strip():
            print(out.stderr[-800:])
print("sequential ms", [round(x, 3) for x in res["0"]], " concurrent ms", [round(x, 3) for x in res["1"]])
