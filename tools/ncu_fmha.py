"""Dev tool: one cfg5-shaped UP launch for an ncu capture of the fused attention kernel
(`ncu --set full -k regex:fmha -c 1 python tools/ncu_fmha.py`)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")
T, heads, S = 8, 4, int(os.environ.get("NCU_FMHA_S", "32768"))
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = (torch.randn((T, heads, S, 128), device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
o = torch.empty((T, 1, S // T, T * heads * 128), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.local_group(T, 2 * (S // T) * T * heads * 128 * 2 + (8 << 20))
comm.attention_a2a(q, k, v, o, 1, heads)
comm.sync()
torch.cuda.synchronize()
comm.close()
print("ok")
