"""Dev tool: one T = 1 GEMM of the bench block (op 'rs': 8192x14336x4096 down projection; 'ag':
8192x4096x28672 gate||up + SwiGLU) timed over 20 calls; run under ncu for the per-launch DRAM
bytes. The raster / L2-hint settings come from TPF_GROUP_M, TPF_GROUP_N, TPF_L2_A, TPF_L2_B.
    python tools/l2_probe.py rs|ag"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2604_24013_b200 as tpf

op = sys.argv[1]
dev = torch.device("cuda:0")
if os.environ.get("PERSIST_MB"):
    # L2 set-aside for persisting (evict_last) lines, cudaLimitPersistingL2CacheSize = 0x06
    import ctypes
    torch.cuda.init()
    rt = ctypes.CDLL("libcudart.so.12")
    mx = ctypes.c_int(0)
    rt.cudaDeviceGetAttribute(ctypes.byref(mx), 108, 0)  # cudaDevAttrMaxPersistingL2CacheSize
    want = min(int(os.environ["PERSIST_MB"]) << 20, mx.value)
    print("persisting L2 set-aside", want >> 20, "MB of max", mx.value >> 20, "MB; rc",
          rt.cudaDeviceSetLimit(6, ctypes.c_size_t(want)))
g = torch.Generator(device=dev).manual_seed(0)
one = tpf.Communicator.create(0, 1, 0)
if op == "rs":
    x = torch.randn((1, 8192, 14336), device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn((14336, 4096), device=dev, generator=g) / 120).to(torch.bfloat16)
    y = torch.empty((1, 8192, 4096), device=dev, dtype=torch.bfloat16)
    fn = lambda: one.gemm_rs(x, w, y)  # noqa: E731
    flops = 2.0 * 8192 * 14336 * 4096
else:
    x = torch.randn((1, 8192, 4096), device=dev, generator=g).to(torch.bfloat16)
    w = (torch.randn((4096, 28672), device=dev, generator=g) / 64).to(torch.bfloat16)
    y = torch.empty((1, 8192, 14336), device=dev, dtype=torch.bfloat16)
    fn = lambda: one.ag_gemm(x, w, y, act=tpf.ACT_SWIGLU)  # noqa: E731
    flops = 2.0 * 8192 * 4096 * 28672
n = int(os.environ.get("PROBE_N", "20"))
for _ in range(3):
    fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(n):
    fn()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"{op} GM={os.environ.get('TPF_GROUP_M', '16')} GN={os.environ.get('TPF_GROUP_N', '0')} "
      f"L2A={os.environ.get('TPF_L2_A', '0')} L2B={os.environ.get('TPF_L2_B', '0')}: {1e3 * ms:.1f} us "
      f"{flops / ms / 1e9:.0f} TF/s", flush=True)
