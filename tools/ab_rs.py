"""Dev tool: A/B two library builds on GEMM-RS / AG-GEMM exposed comm (local group),
alternating processes. python tools/ab_rs.py LIB_A LIB_B [rounds]"""
import json
import os
import subprocess
import sys

CODE = r'''
import json, os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_2604_24013_b200 as tpf
dev = torch.device("cuda:0")
def one(fn):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
res = {}
for name, T, S, K, N, op in (("cfg2_rs_T8", 8, 8192, 14336, 4096, "rs"), ("cfg3_rs_T4", 4, 16384, 8192, 8192, "rs"),
                             ("cfg3_rs_T8", 8, 16384, 8192, 8192, "rs"), ("cfg2_ag_T8", 8, 8192, 4096, 28672, "ag")):
    g = torch.Generator(device=dev).manual_seed(0)
    if op == "rs":
        x = torch.randn((T, 1, S, K // T), device=dev, generator=g).to(torch.bfloat16)
        w = (torch.randn((T, K // T, N), device=dev, generator=g) / 64).to(torch.bfloat16)
        y = torch.empty((T, 1, S // T, N), device=dev, dtype=torch.bfloat16)
        comm = tpf.Communicator.local_group(T, tpf.sym_bytes_rs(T, 1, S, K // T, N, 1, tpf.BF16))
        fn = lambda: comm.gemm_rs(x, w, y, kind=tpf.RING, wire=tpf.BF16)
    else:
        x = torch.randn((T, 1, S // T, K), device=dev, generator=g).to(torch.bfloat16)
        w = (torch.randn((T, K, N // T), device=dev, generator=g) / 64).to(torch.bfloat16)
        y = torch.empty((T, 1, S, N // T), device=dev, dtype=torch.bfloat16)
        comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ag(T, 1, S, K, N // T))
        fn = lambda: comm.ag_gemm(x, w, y)
    for _ in range(2): fn()
    f, c = [], []
    for _ in range(7):
        f.append(one(fn)); comm.set_compute_only(True); c.append(one(fn)); comm.set_compute_only(False)
    comm.sync(); comm.close()
    res[name] = [round(statistics.median(f), 4), round(1e3 * (statistics.median(f) - statistics.median(c)), 1)]
print(json.dumps(res))
'''

libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
for r in range(rounds):
    for l in libs:
        env = dict(os.environ, TPF_LIB_PATH=os.path.abspath(l))
        out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
        print(os.path.basename(os.path.dirname(l)) or l, out.stdout.strip().splitlines()[-1] if out.stdout else out.stderr[-500:],
              flush=True)
