"""Small invocations of every fused operator, for compute-sanitizer (memcheck / synccheck /
racecheck). python tools/sanitize_smoke.py; compute-sanitizer --tool memcheck python ..."""
import os
import sys

sys.path.insert(0, os.getcwd())
os.environ.setdefault("TPF_TIMEOUT_MS", "600000")
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")
T, B, S, K, N = 2, 1, 512, 256, 512
g = torch.Generator(device=dev).manual_seed(0)
r = lambda *shape: (torch.randn(shape, device=dev, generator=g) / 8).to(torch.bfloat16)  # noqa: E731
comm = tpf.Communicator.local_group(T, max(tpf.sym_bytes_ag(T, B, S, K, N // T), tpf.sym_bytes_rs(T, B, S, K // T, N, 1),
                                           tpf.sym_bytes_ulysses(T, B, 4, S, 128), tpf.sym_bytes_dp_ag(T, K, N // T)))
x = r(T, B, S // T, K)
w = r(T, K, N // T)
y = torch.empty((T, B, S, N // T), device=dev)
comm.ag_gemm(x, w, y)
xr = r(T, B, S, K // T)
wr = r(T, K // T, N)
yr = torch.empty((T, B, S // T, N), device=dev)
for kind in (tpf.RING, tpf.PAIRWISE, tpf.CIRCULAR):
    comm.gemm_rs(xr, wr, yr, kind=kind)
q = r(T, B * 2, S, 128)
o = torch.empty((T, B, S // T, T * 2 * 128), device=dev, dtype=torch.bfloat16)
comm.attention_a2a(q, q, q, o, B, 2)
qs = r(T, B * 4, S // T, 128)
ou = torch.empty((T, B, S // T, 4 * 128), device=dev, dtype=torch.bfloat16)
comm.ulysses_attention(qs, qs, qs, ou, B, 4)
wo = r(T, 2 * 128, 256)
oq = torch.empty((T, B, S // T, 256), device=dev)
comm.query_split_attention(q, q, q, wo, oq, B, 2)
X = r(T, 256, K)
dY = r(T, 256, N)
dW = torch.empty((T, K // T, N), device=dev)
comm.dp_grad_rs(X, dY, dW)
comm.sync()
comm.close()
a, b = r(256, 128), r(128, 256)
c = torch.empty((256, 256), device=dev)
tpf.gemm(a, b, c)
torch.cuda.synchronize()
print("sanitize smoke ok")
