"""Dev tool: UP (fused attention + all-to-all) timing on one GPU (local group)."""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2604_24013_b200 as tpf
dev = torch.device("cuda:0")
for T, heads, S in ((8, 4, 32768), (8, 4, 8192), (1, 32, 8192)):
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
    fl = 4.0 * T * heads * S * S * 128
    print(f"UP T={T} heads/rank={heads} S={S}: {t:.3f} ms  {fl / t / 1e9:.0f} TF/s", flush=True)
    comm.close()
