"""Dev tool: A/B two library builds on the per-GPU TP = 8 (AB_T) fused ops (virtual peers, cfg2 and
cfg3 shapes, AG-GEMM and GEMM-RS), alternating processes to cancel power-cap drift. Prints
the median us per call (20 back-to-back calls) for each build.
    python tools/ab_lib.py LIB_A LIB_B [rounds]
A spec may carry environment settings: 'lib.so@TPF_AG_SPLIT=0@TPF_X=1'. AB_ONLY=cfg4 runs only
the cfg4 DP rows."""
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
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / n
res = {}
T = int(os.environ.get("AB_T", "8"))
CFGS = (("cfg2", 8192, 4096, 28672, 14336, 4096), ("cfg3", 16384, 8192, 10240, 8192, 8192))
for cfg, S, K_ag, N_ag, K_rs, N_rs in (() if os.environ.get("AB_ONLY") == "cfg4" else CFGS):
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn((1, S // T, K_ag), device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn((K_ag, N_ag // T), device=dev, generator=g) / 64).to(torch.bfloat16)
    y = torch.empty((1, S, N_ag // T), device=dev, dtype=torch.bfloat16)
    xr = torch.randn((1, S, K_rs // T), device=dev, generator=g).to(torch.bfloat16)
    wr = (torch.randn((K_rs // T, N_rs), device=dev, generator=g) / 64).to(torch.bfloat16)
    yr = torch.empty((1, S // T, N_rs), device=dev, dtype=torch.bfloat16)
    xg = torch.randn((S, K_ag), device=dev, generator=g).to(torch.bfloat16)
    yg = torch.empty((S, N_ag // T), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, K_ag, N_ag // T),
                                                 tpf.sym_bytes_rs(T, 1, S, K_rs // T, N_rs, 1, tpf.BF16)))
    res[cfg + "_ag"] = loop(lambda: comm.ag_gemm(x, w, y))
    res[cfg + "_rs"] = loop(lambda: comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=tpf.BF16))
    if T % 2 == 0:
        res[cfg + "_rs_pw"] = loop(lambda: comm.gemm_rs(xr, wr, yr, kind=tpf.PAIRWISE, wire=tpf.BF16))
    res[cfg + "_rs_circ"] = loop(lambda: comm.gemm_rs(xr, wr, yr, kind=tpf.CIRCULAR, wire=tpf.BF16))
    res[cfg + "_ag_gemm"] = loop(lambda: tpf.gemm(xg, w, yg))
    comm.set_compute_only(True)
    res[cfg + "_ag_co"] = loop(lambda: comm.ag_gemm(x, w, y))
    comm.set_compute_only(False)
    comm.close()
if T == 8:
    # cfg4 DP per GPU: parameter AG fused into the forward GEMM (gather_b) and gradient RS
    M, K, N = 4096, 2048, 8192
    g = torch.Generator(device=dev).manual_seed(1)
    X = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
    dY = (torch.randn((M, N), device=dev, generator=g) / 64).to(torch.bfloat16)
    dW = torch.empty((K // T, N), device=dev, dtype=torch.bfloat16)
    Wr = (torch.randn((N // T, K), device=dev, generator=g) / 45).to(torch.bfloat16)
    out = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_rs(T, 1, K, M, N, 1, tpf.BF16),
                                                 tpf.sym_bytes_dp_ag(T, K, N // T)))
    res["cfg4_param_ag"] = loop(lambda: comm.dp_param_ag_gemm(X, Wr, out))
    res["cfg4_grad_rs"] = loop(lambda: comm.dp_grad_rs(X, dY, dW, kind=tpf.RING, wire=tpf.BF16))
    res["cfg4_grad_rs_pw"] = loop(lambda: comm.dp_grad_rs(X, dY, dW, kind=tpf.PAIRWISE, wire=tpf.BF16))
    comm.close()
print(json.dumps(res))
'''
libs = sys.argv[1:3]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 4
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
            print(lib, "failed:", out.stderr[-1500:], flush=True)
for lib in libs:
    if res[lib]:
        keys = res[lib][0].keys()
        print(lib, {k: round(statistics.median(r[k] for r in res[lib]), 1) for k in keys},
              "runs", [{k: round(v) for k, v in r.items()} for r in res[lib]])
