"""Dev tool: one fused AG-GEMM and one fused GEMM-RS of a TP group's rank 0 with virtual peers
(cfg2 shapes), for an ncu capture of the protocol at full-GPU scale.
    python tools/ncu_virtual_ops.py T [co]   (co: also one compute-only AG-GEMM, for a side-by-side)
Profile with ncu -s 6 -c 2 (the fourth AG-GEMM and GEMM-RS)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
S, D, F = 8192, 4096, 14336
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
x = torch.randn((1, S // T, D), device=dev, generator=g).to(torch.bfloat16)
w = (torch.randn((D, 2 * F // T), device=dev, generator=g) / 64).to(torch.bfloat16)
y = torch.empty((1, S, 2 * F // T), device=dev, dtype=torch.bfloat16)
xr = torch.randn((1, S, F // T), device=dev, generator=g).to(torch.bfloat16)
wr = (torch.randn((F // T, D), device=dev, generator=g) / 64).to(torch.bfloat16)
yr = torch.empty((1, S // T, D), device=dev, dtype=torch.bfloat16)
comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, D, 2 * F // T),
                                             tpf.sym_bytes_rs(T, 1, S, F // T, D, 1, tpf.BF16)))
# four calls of each: profile the last pair (ncu -s 6 -c 2), at steady state. Replays restore
# memory to the state before the profiled launch, so the ring's step-to-step waits are real in
# the capture.
for _ in range(4):
    comm.ag_gemm(x, w, y)
    comm.gemm_rs(xr, wr, yr, kind=tpf.RING, wire=tpf.BF16)
if len(sys.argv) > 2 and sys.argv[2] == "co":
    comm.set_compute_only(True)
    comm.ag_gemm(x, w, y)
    comm.set_compute_only(False)
torch.cuda.synchronize()
comm.close()
print("ok")
