import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2604_24013_b200 as tpf
dev = torch.device("cuda:0")
T, S, K, N = int(sys.argv[1]), 16384, 8192, 10240
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn((T, 1, S // T, K), device=dev, generator=g).to(torch.bfloat16)
w = (torch.randn((T, K, N // T), device=dev, generator=g) / 90).to(torch.bfloat16)
y = torch.empty((T, 1, S, N // T), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ag(T, 1, S, K, N // T))
def one():
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record(); comm.ag_gemm(x, w, y); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
def b2b(n=5):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(n): comm.ag_gemm(x, w, y)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for co in (False, True):
    comm.set_compute_only(co)
    for _ in range(3): one()
    print("compute_only" if co else "fused", "isolated", [round(one(), 3) for _ in range(4)], "b2b", [round(b2b(), 3) for _ in range(3)], flush=True)
comm.sync(); comm.close()
