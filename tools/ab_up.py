"""Dev tool: A/B library builds (TPF_LIB_PATH) on the UP attention (cfg5 T = 8 local group and a
per-GPU shape), alternating fresh processes.   python tools/ab_up.py LIB_A LIB_B ... [--rounds N]
A spec may carry environment settings: 'lib.so@TPF_FMHA_PAIR=0'."""
import os
import statistics
import subprocess
import sys

CODE = r'''
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2604_24013_b200 as tpf
dev = torch.device("cuda:0")
out = []
for T, heads, S in ((8, 4, 32768), (1, 32, 8192)):
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v = (torch.randn((T, heads, S, 128), device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
    o = torch.empty((T, 1, S // T, T * heads * 128), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.local_group(T, 2 * (S // T) * T * heads * 128 * 2 + (8 << 20))
    for _ in range(2): comm.attention_a2a(q, k, v, o, 1, heads)
    comm.sync(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3): comm.attention_a2a(q, k, v, o, 1, heads)
    e1.record(); torch.cuda.synchronize(); comm.sync()
    t = e0.elapsed_time(e1) / 3
    out.append(4.0 * T * heads * S * S * 128 / t / 1e9)
    comm.close()
print(" ".join(f"{x:.0f}" for x in out))
'''
args = [a for a in sys.argv[1:] if not a.startswith("--")]
rounds = int(sys.argv[sys.argv.index("--rounds") + 1]) if "--rounds" in sys.argv else 3
args = [a for a in args if not a.isdigit()]
res = {a: [] for a in args}
for _ in range(rounds):
    for lib in args:
        path, *kvs = lib.split("@")  # 'lib.so@ENV=V' runs the build under an environment setting
        env = dict(os.environ, TPF_LIB_PATH=os.path.abspath(path))
        env.update(kv.split("=", 1) for kv in kvs)
        r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=900)
        try:
            res[lib].append([float(x) for x in r.stdout.strip().splitlines()[-1].split()])
        except Exception:
            print(lib, "failed", r.stderr[-800:])
for lib, v in res.items():
    if v:
        print(lib, "TF/s cfg5 T8 / T1 S8192:", [round(statistics.median(c)) for c in zip(*v)], "runs", v)
