"""Dev tool: A/B settings on the per-GPU cfg4 DP ops alone (virtual peers, TP = 8 ranks), in
alternating fresh processes.   python tools/ab_dp.py 'lib.so@ENV=V' 'lib.so' [rounds]"""
import json
import os
import statistics
import subprocess
import sys

CODE = r'''
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2604_24013_b200 as tpf
dev = torch.device("cuda:0")
def loop(fn, n=20):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / n
T, M, K, N = 8, 4096, 2048, 8192
g = torch.Generator(device=dev).manual_seed(1)
X = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
dY = (torch.randn((M, N), device=dev, generator=g) / 64).to(torch.bfloat16)
dW = torch.empty((K // T, N), device=dev, dtype=torch.bfloat16)
Wr = (torch.randn((N // T, K), device=dev, generator=g) / 45).to(torch.bfloat16)
out = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_rs(T, 1, K, M, N, 1, tpf.BF16), tpf.sym_bytes_dp_ag(T, K, N // T)))
res = {"param_ag": min(loop(lambda: comm.dp_param_ag_gemm(X, Wr, out)) for _ in range(3)),
       "grad_rs": min(loop(lambda: comm.dp_grad_rs(X, dY, dW, kind=tpf.RING, wire=tpf.BF16)) for _ in range(3))}
comm.close()
print(json.dumps(res))
'''
libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 6
res = {lib: [] for lib in libs}
for _ in range(rounds):
    for lib in libs:
        path, *kvs = lib.split("@")
        env = dict(os.environ, TPF_LIB_PATH=os.path.abspath(path))
        env.update(kv.split("=", 1) for kv in kvs)
        out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
        try:
            res[lib].append(json.loads(out.stdout.strip().splitlines()[-1]))
        except Exception:
            print(lib, "failed:", out.stderr[-800:], flush=True)
for lib in libs:
    if res[lib]:
        print(lib, {k: round(statistics.median(r[k] for r in res[lib]), 1) for k in res[lib][0]},
              "runs", [{k: round(v) for k, v in r.items()} for r in res[lib]])
