"""Per-GPU UP attention of one rank of a real TP group (virtual peers): the fused attention
kernel on the whole GPU (148 CTAs) for one rank's work, as on an NVSwitch box.
    python tools/perf_up_virtual.py [T] [heads_per_rank] [S]"""
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

T, heads, S = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else ("8", "4", "32768")))
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = (torch.randn((heads, S, 128), device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
o = torch.empty((1, S // T, T * heads * 128), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.virtual_group(T, tpf.sym_bytes_ulysses(T, 1, T * heads, S, 128))
for _ in range(2):
    comm.attention_a2a(q, k, v, o, 1, heads)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    comm.attention_a2a(q, k, v, o, 1, heads)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
comm.close()
ms = statistics.median(ts)
fl = 4.0 * heads * S * S * 128
items = T * heads * ((S // T // 128 + 1) // 2)
print(f"virtual T={T} heads/rank={heads} S={S}: {ms:.3f} ms {fl / ms / 1e9:.0f} TF/s  items={items} "
      f"rounds on 148 CTAs={items / 148:.2f}")
