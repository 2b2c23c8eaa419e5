"""Dev tool: one launch of each auxiliary kernel, for an ncu --set full capture (every
kernel's capture): the flag-wait kernels (wait_flags, wait_flags2), the parity-selected copy
(copy_by_parity), the unfused attention's softmax (softmax_rows, head_dim 64 fallback), the
Ulysses push kernel, the unfused SwiGLU and the split-group GEMM kernel.
    python tools/ncu_aux.py"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
T, batch, heads = 4, 1, 8
# unfused attention (head_dim 64): QK^T GEMM, softmax_rows, P.V GEMM with push, wait_flags
S, Dh = 2048, 64
q, k, v = (torch.randn((T, batch * heads // T, S, Dh), device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
out = torch.empty((T, batch, S // T, heads * Dh), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ulysses(T, batch, heads, S, Dh))
comm.attention_a2a(q, k, v, out, batch, heads // T)
comm.sync()
# Ulysses first all-to-all: ulysses_push, wait_flags2, copy_by_parity
S2, Dh2 = 4096, 128
xs = [torch.randn((T, batch * heads, S2 // T, Dh2), device=dev, generator=g).to(torch.bfloat16) for _ in range(3)]
outs = [torch.empty((T, batch * heads // T, S2, Dh2), device=dev, dtype=torch.bfloat16) for _ in range(3)]
comm2 = tpf.Communicator.local_group(T, tpf.sym_bytes_ulysses(T, batch, heads, S2, Dh2))
comm2.ulysses_a2a(*xs, *outs, batch, heads)
comm2.sync()
# unfused SwiGLU
gu = torch.randn((8192, 2 * 1792), device=dev, generator=g).to(torch.bfloat16)
act = torch.empty((8192, 1792), device=dev, dtype=torch.bfloat16)
tpf.swiglu(gu, act)
# split group: the per-rank GEMM-RS of 4 ranks as one grid
Ss, K, N = 4096, 4096, 4096
xr = torch.randn((T, 1, Ss, K // T), device=dev, generator=g).to(torch.bfloat16)
wr = (torch.randn((T, K // T, N), device=dev, generator=g) / 32).to(torch.bfloat16)
yr = torch.empty((T, 1, Ss // T, N), device=dev, dtype=torch.bfloat16)
comms = tpf.Communicator.split_group(T, tpf.sym_bytes_rs(T, 1, Ss, K // T, N, 1, tpf.BF16))
for r in range(T):
    comms[r].gemm_rs(xr[r], wr[r], yr[r], wire=tpf.BF16)
for c in comms:
    c.sync()
torch.cuda.synchronize()
print("ok")
