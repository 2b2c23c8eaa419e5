"""The one-process-per-rank path on a real GPU: two processes on cuda:0, CUDA-IPC handles
exchanged over torch.distributed (gloo), peers opened, then fused AG-GEMM / GEMM-RS calls
in compute-only mode (the same kernels and tile schedule with every peer wait and wire
transfer disabled). Two processes' kernels that waited on one another must not share one
GPU (they are not guaranteed to run concurrently), so the cross-process data path itself
is covered by the one-launch local group; this test covers the multi-process plumbing the
N > 1 bench runs through (Communicator.from_process_group, tpf_comm_open_peers, per-process
device epochs) and checks the slices compute-only mode does compute."""
import os
import socket
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_24013_b200 as tpf
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        T, S, K, N = world, 512, 256, 512
        sl, nl = S // T, N // T
        need = max(tpf.sym_bytes_ag(T, 1, S, K, nl), tpf.sym_bytes_rs(T, 1, S, K // T, N))
        comm = tpf.Communicator.from_process_group(need)
        assert (comm.rank, comm.world, comm.is_local_group) == (rank, world, False)
        comm.set_compute_only(True)
        g = torch.Generator(device=dev).manual_seed(100 + rank)
        # AG-GEMM: at step 0 every rank computes its own sequence chunk into its own rows
        x = torch.randn((1, sl, K), device=dev, generator=g).to(torch.bfloat16)
        w = (torch.randn((K, nl), device=dev, generator=g) / 16).to(torch.bfloat16)
        out = torch.full((1, S, nl), float("nan"), device=dev)
        ref = torch.empty((sl, nl), device=dev)
        for _ in range(3):  # back-to-back calls advance the device epoch
            comm.ag_gemm(x, w, out)
        comm.sync()
        tpf.gemm(x[0], w, ref)
        torch.cuda.synchronize()
        assert torch.equal(out[0, rank * sl:(rank + 1) * sl], ref), "AG own slice"
        # GEMM-RS: compute-only stores every step's partial into the output, and tiles of
        # different steps race, so each 16-B store (4 fp32 columns of a row) holds the
        # partial of one of the T slices
        xr = torch.randn((1, S, K // T), device=dev, generator=g).to(torch.bfloat16)
        wr = (torch.randn((K // T, N), device=dev, generator=g) / 16).to(torch.bfloat16)
        yr = torch.full((1, sl, N), float("nan"), device=dev)
        for kind in (tpf.RING, tpf.PAIRWISE, tpf.CIRCULAR):
            comm.gemm_rs(xr, wr, yr, kind=kind)
        comm.sync()
        parts = []
        for l in range(T):
            pr = torch.empty((sl, N), device=dev)
            tpf.gemm(xr[0, l * sl:(l + 1) * sl].contiguous(), wr, pr)
            parts.append(pr)
        torch.cuda.synchronize()
        eq = torch.stack([yr[0] == pr for pr in parts])  # (T, sl, N)
        assert bool(eq.view(T, sl, N // 4, 4).all(-1).any(0).all()), "RS compute-only stores"
        comm.close()
        dist.barrier()
        q.put((rank, "ok"))
    except Exception:
        import traceback
        tb = traceback.format_exc()
        print(f"rank {rank}:\n{tb}", file=sys.stderr, flush=True)
        q.put((rank, tb))
    finally:
        dist.destroy_process_group()


def test_two_processes_share_ipc_heaps_compute_only():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    bad = {r: v for r, v in results.items() if v != "ok"}
    assert not bad, bad
