"""Dev tool: one cfg5-shaped Ulysses first all-to-all for an ncu capture of the push kernel
(`ncu --set full -k regex:ulysses -c 1 python tools/ncu_ulysses.py`)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

dev = torch.device("cuda:0")
T, H, S, Dh = 8, 32, 32768, 128
g = torch.Generator(device=dev).manual_seed(0)
xs = [torch.randn((T, H, S // T, Dh), device=dev, generator=g).to(torch.bfloat16) for _ in range(3)]
outs = [torch.empty((T, H // T, S, Dh), device=dev, dtype=torch.bfloat16) for _ in range(3)]
comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ulysses(T, 1, H, S, Dh))
comm.ulysses_a2a(*xs, *outs, 1, H)
comm.sync()
torch.cuda.synchronize()
comm.close()
print("ok")
