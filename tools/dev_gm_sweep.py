import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import paper_2604_24013_b200 as tpf
T = int(sys.argv[1])
S, K, N = 8192, 4096, 28672
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn((1, S // T, K), device=dev, generator=g).to(torch.bfloat16)
w = (torch.randn((K, N // T), device=dev, generator=g) / 64).to(torch.bfloat16)
y = torch.empty((1, S, N // T), device=dev, dtype=torch.bfloat16)
xg = torch.randn((S, K), device=dev, generator=g).to(torch.bfloat16)
yg = torch.empty((S, N // T), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.virtual_group(T, tpf.sym_bytes_ag(T, 1, S, K, N // T))
def one(fn):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record(); fn(); e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)
for _ in range(3): comm.ag_gemm(x, w, y); tpf.gemm(xg, w, yg)
f, c, p = [], [], []
for _ in range(9):
    f.append(one(lambda: comm.ag_gemm(x, w, y)))
    comm.set_compute_only(True); c.append(one(lambda: comm.ag_gemm(x, w, y))); comm.set_compute_only(False)
    p.append(one(lambda: tpf.gemm(xg, w, yg)))
print(os.environ.get("TPF_GROUP_M", "16"), T, "fused %.4f co %.4f plain %.4f" % (statistics.median(f), statistics.median(c), statistics.median(p)))
comm.close()
