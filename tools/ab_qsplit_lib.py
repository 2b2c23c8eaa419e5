"""Dev tool: query_split_attention (concurrent attention + GEMM-RS) timed under several
library builds, alternating processes (AB_WIRE=f32 for the fp32 wire and output).
python tools/ab_qsplit_lib.py LIB..."""
import os
import statistics
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
f32 = os.environ.get("AB_WIRE", "bf16") == "f32"
out = torch.empty((T, 1, S // T, D), device=dev, dtype=torch.float32 if f32 else torch.bfloat16)
wire = tpf.F32 if f32 else tpf.BF16
comm = tpf.Communicator.local_group(T, tpf.sym_bytes_rs(T, 1, S, h * 128, D, 1, wire) + (1 << 22))
fn = lambda: comm.query_split_attention(q, k, v, w, out, 1, h, wire=wire)
for _ in range(3): fn()
torch.cuda.synchronize()
ts = []
for _ in range(7):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
comm.sync(); comm.close()
print(statistics.median(ts))
'''
libs = [a for a in sys.argv[1:] if a.endswith(".so")]
shape = ["4", "8192", "8", "4096"]
res = {lib: [] for lib in libs}
for _ in range(3):
    for lib in libs:
        env = dict(os.environ, TPF_LIB_PATH=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", CODE] + shape, env=env, capture_output=True, text=True, timeout=300)
        res[lib].append(float(out.stdout.strip().splitlines()[-1]) if out.stdout.strip() else -1.0)
        if not out.stdout.strip():
            print(lib, out.stderr[-800:])
for lib in libs:
    print(lib, "median ms", round(statistics.median(res[lib]), 3), [round(x, 3) for x in res[lib]])
