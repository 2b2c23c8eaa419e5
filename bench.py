#!/usr/bin/env python
"""Benchmark: Llama-3-8B TP-SP MLP block, seq 8192, TP = number of GPUs (BASELINE cfg 2).

One step = one forward of the block through this library's fused ops:
    AG-GEMM   hidden = all_gather_seq(x) @ W_gate||up[r]     (column_parallel_forward)
    SwiGLU    act    = silu(gate) * up
    GEMM-RS   y      = reduce_scatter_seq(act @ W_down[r])   (row_parallel_forward)
x: (1, 8192/T, 4096) bf16 per rank, W_gate||up: (4096, 28672/T), W_down: (14336/T, 4096).
At N=1 (T=1) both ops are the degenerate plain GEMM (collectives.cpp:242,379).

Prints ONE JSON line (rank 0). `value` = whole-job TFLOP/s with inputs resident in HBM;
`e2e` = the same through the C-ABI calls with pinned HOST input/output and the copies
inside the timed region; `roofline` for the dominant kernel (the AG-GEMM launch), timed
live with CUDA events on its stream; `cpu_baseline` = the reference's own CPU code
(oracle/_ref, compiled from /root/reference) on a bounded sample, timed on this host.

At N > 1 (one rank per GPU, NCCL for plumbing, CUDA-IPC symmetric heaps for the data) the
line adds, per op, the plain per-rank GEMM of the same shapes (exposed comm = fused - plain,
acceptance C6), the measured tail from a device trace (acceptance C4), and the NCCL
all-gather / reduce-scatter + cuBLAS non-overlapped baseline run in the same job. At N = 1 it
adds one GPU of a TP = 8 group at full scale (virtual peers) with the same comparisons.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--dry-run]

`--gpus N` without a torchrun environment launches the N ranks itself (torch.distributed.run,
127.0.0.1); under torchrun WORLD_SIZE must equal N. `--dry-run` exercises only the launcher
and rank plumbing (gloo, no GPU).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

D_MODEL, FFN, SEQ = 4096, 14336, 8192
WORKLOAD = "Llama-3-8B TP-SP MLP block (AG-GEMM gate||up + fused SwiGLU -> GEMM-RS down), seq 8192"
METRIC = "AG-GEMM/GEMM-RS TFLOP/s & exposed-comm us at TP=2/4/8; % of roofline"


def block_flops(tokens: int) -> float:
    return 2.0 * tokens * D_MODEL * (2 * FFN) + 2.0 * tokens * FFN * D_MODEL


def peaks():
    p = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "src": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("bf16_tflops", "bf16_tflops_sustained", "hbm_gbs") if k in m})
        p["src"] = "measured"
    return p


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.samples, self.proc, self.t0, self.t1 = [], None, None, None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def wait_ready(self, timeout=5.0):
        """Block until nvidia-smi has produced its first sample (its start-up takes
        ~0.1-0.5 s), so the timed region that follows is actually sampled."""
        t_end = time.time() + timeout
        while self.proc and not self.samples and time.time() < t_end:
            time.sleep(0.01)

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        rows = [s for t, s in self.samples if self.t0 and self.t1 and self.t0 - 0.02 <= t <= self.t1 + 0.02]
        window = "timed_region"
        if not rows:
            rows, window = [s for _, s in self.samples], "whole_run"
        mhz, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            f = [v.strip() for v in r.split(",")]
            if len(f) < 6:
                continue
            try:
                mhz.append(float(f[0]))
                maxes.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not mhz:
            return None
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": max(maxes), "reasons": sorted(reasons),
                "samples": len(mhz), "window": window}


# ------------------------------------------------------------- CPU reference
def cpu_reference_sample(threads: int, tokens_per_rank: int, reps: int = 1):
    """The reference's own CPU path (oracle/_ref = /root/reference/proj/src compiled
    in place) on a bounded sample of the same block: `threads` simulated TP ranks (one
    worker thread per rank, fabric.hpp:196-213), tokens_per_rank * threads tokens.
    Returns per-repetition records."""
    from oracle_lib import Reference, have_reference
    if not have_reference():
        return None
    R = Reference()
    t = threads
    s_cpu = tokens_per_rank * t
    ag, rs = R.time_ops(t, 1, s_cpu, D_MODEL, 2 * FFN, FFN, D_MODEL, reps)
    return [{"tokens": s_cpu, "ranks": t, "seconds": a + b, "ag_seconds": a, "rs_seconds": b,
             "tflops": block_flops(s_cpu) / (a + b) / 1e12} for a, b in zip(ag, rs)]


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    nproc = os.cpu_count() or 1
    t = max(1, min(8, nproc))
    recs = cpu_reference_sample(t, 1, args.warmup + args.steps)
    if recs is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtpfuse_ref.so not built"}))
        return
    per_step = recs[args.warmup:]
    secs = sum(r["seconds"] for r in per_step)
    flops = sum(block_flops(r["tokens"]) for r in per_step)
    value = flops / secs / 1e12
    sample = (f"{per_step[0]['tokens']} tokens of the block per step, {t} simulated TP ranks, one thread "
              f"each (reference column_parallel_forward + row_parallel_forward, fp64), host nproc={nproc}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / len(per_step), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference randint recipe)",
        "config": {"workload": WORKLOAD, "tp": world, "seq_len": SEQ, "d_model": D_MODEL, "ffn": FFN,
                   "global_batch": 1, "parallelism": f"tp{world}-sp (reference: {t} rank threads)"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": t, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ------------------------------------------------------------------ our arm
def _events(n, k=3):
    import torch
    return [[torch.cuda.Event(enable_timing=True) for _ in range(k)] for _ in range(n)]


def _timed_calls(fn, stream, n):
    """n back-to-back calls between two events on the launch stream: device ms per call."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def traced_tail(comm, fn, dev):
    """Measured no_tail_check (costmodel.cpp:163-176 on a %globaltimer timeline):
    one traced call; per rank, the last peer-flag publication minus the end of the last GEMM
    tile. Returns the max tail in us over this process's ranks."""
    import torch

    from paper_2604_24013_b200 import trace
    buf = trace.alloc(300000, dev)
    torch.cuda.synchronize(dev)
    comm.set_trace(buf)
    fn()
    comm.sync()
    comm.set_trace(None)
    summ = trace.summarize(trace.decode(buf))
    return max((v["tail_us"] for v in summ.values()), default=0.0)



def e2e_pipeline(torch, n, x_host, y_host, x_dev, y_dev, compute, stream, dev, barrier=lambda: None):
    """The e2e timed region: n steps, each copying its input from pinned host memory
    (x_host[i % nbuf] -> x_dev) on one stream, running compute(x_dev[b], y_dev[b]) on the
    compute stream and copying the result back (y_dev[b] -> y_host[b]) on another, with
    nbuf-deep double buffering so step i+1's H2D and step i-1's D2H overlap step i's kernels.
    Returns ms per step (first H2D start to last D2H end). Tested for correct ordering in
    tests/test_gpu_e2e.py."""
    nbuf = len(x_host)
    s_in = torch.cuda.Stream(dev)
    s_out = torch.cuda.Stream(dev)
    ev_in = [torch.cuda.Event() for _ in range(n)]
    ev_done = [torch.cuda.Event() for _ in range(n)]
    ev_out = [torch.cuda.Event() for _ in range(n)]
    barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_in)
    stream.wait_stream(s_in)
    s_out.wait_stream(s_in)
    for i in range(n):
        b = i % nbuf
        with torch.cuda.stream(s_in):
            if i >= nbuf:
                s_in.wait_event(ev_done[i - nbuf])  # x_dev[b] consumed by step i-nbuf
            x_dev[b].copy_(x_host[b], non_blocking=True)
            ev_in[i].record(s_in)
        stream.wait_event(ev_in[i])
        if i >= nbuf:
            stream.wait_event(ev_out[i - nbuf])  # y_dev[b] drained by step i-nbuf's D2H
        compute(x_dev[b], y_dev[b])
        ev_done[i].record(stream)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_done[i])
            y_host[b].copy_(y_dev[b], non_blocking=True)
            ev_out[i].record(s_out)
    s_out.wait_stream(stream)
    e1.record(s_out)
    torch.cuda.synchronize(dev)
    barrier()
    return e0.elapsed_time(e1) / n

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2604_24013_b200 as tpf

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    T = world
    S_l, F_l = SEQ // T, FFN // T
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    x = torch.randn((1, S_l, D_MODEL), device=dev, generator=g).to(torch.bfloat16)
    w_gate = (torch.randn((D_MODEL, F_l), device=dev, generator=g) / D_MODEL ** 0.5).to(torch.bfloat16)
    w_up = (torch.randn((D_MODEL, F_l), device=dev, generator=g) / D_MODEL ** 0.5).to(torch.bfloat16)
    w_gu = tpf.interleave_gate_up(w_gate, w_up).contiguous()  # fused-SwiGLU shard layout
    w_dn = (torch.randn((F_l, D_MODEL), device=dev, generator=g) / FFN ** 0.5).to(torch.bfloat16)
    act = torch.empty((1, SEQ, F_l), device=dev, dtype=torch.bfloat16)
    y = torch.empty((1, S_l, D_MODEL), device=dev, dtype=torch.bfloat16)
    stream = torch.cuda.current_stream(dev)

    # T == 1 runs through the same communicator API (degenerate group: plain GEMMs).
    need = max(tpf.sym_bytes_ag(T, 1, SEQ, D_MODEL, 2 * F_l, 1),
               tpf.sym_bytes_rs(T, 1, SEQ, F_l, D_MODEL, 1, tpf.BF16))
    comm = tpf.Communicator.from_process_group(need) if T > 1 else tpf.Communicator.create(0, 1, need)

    def ag(xin=x):
        comm.ag_gemm(xin, w_gu, act, act=tpf.ACT_SWIGLU, stream=stream)

    def rs(yout=y):
        comm.gemm_rs(act, w_dn, yout, kind=tpf.RING, wire=tpf.BF16, stream=stream)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up
    for _ in range(args.warmup):
        ag(); rs()
    comm.sync(stream)
    torch.cuda.synchronize(dev)

    # ---- timed region (device-resident inputs); per-kernel events on the launch stream
    sampler = ClockSampler(local_rank) if rank == 0 else None
    if sampler:
        sampler.wait_ready()
    barrier()
    # keep the GPU busy while sampling settles; every rank runs these (the fused ops are
    # collective: a call only rank 0 made would wait on peers that never join it)
    for _ in range(max(3, args.warmup)):
        ag(); rs()
    n = args.steps
    ev = _events(n)
    barrier()
    torch.cuda.synchronize(dev)
    if sampler:
        sampler.mark_start()
    for i in range(n):
        ev[i][0].record(stream)
        ag()
        ev[i][1].record(stream)
        rs()
        ev[i][2].record(stream)
    torch.cuda.synchronize(dev)
    if sampler:
        sampler.mark_end()
    barrier()
    comm.sync(stream)
    total_ms = ev[0][0].elapsed_time(ev[-1][2])
    ag_ms = sum(e[0].elapsed_time(e[1]) for e in ev) / n
    rs_ms = sum(e[1].elapsed_time(e[2]) for e in ev) / n
    ms_step = max_over_ranks(total_ms / n)
    ag_ms, rs_ms = max_over_ranks(ag_ms), max_over_ranks(rs_ms)
    clocks = sampler.stop() if sampler else None
    flops_step = block_flops(SEQ)  # whole job
    value = flops_step / (ms_step * 1e-3) / 1e12

    # ---- exposed communication (acceptance C6, acceptance_test.cpp:334-366; paper overhead =
    # e2e - compute): the fused op against the PLAIN per-rank GEMM of the same
    # shapes (T = 1 tcgen05 kernel, no collective, same fused SwiGLU epilogue), max over ranks.
    # At N = 1 the ops ARE the plain GEMMs.
    if T > 1:
        one = tpf.Communicator.create(0, 1, 0)
        xg = torch.randn((1, SEQ, D_MODEL), device=dev, generator=g).to(torch.bfloat16)
        yg = torch.empty((1, SEQ, D_MODEL), device=dev, dtype=torch.bfloat16)
        p_ag = lambda: one.ag_gemm(xg, w_gu, act, act=tpf.ACT_SWIGLU, stream=stream)  # noqa: E731
        p_rs = lambda: one.gemm_rs(act, w_dn, yg, stream=stream)  # noqa: E731
        for _ in range(2):
            p_ag(); p_rs()
        plain_ag = max_over_ranks(_timed_calls(p_ag, stream, n))
        plain_rs = max_over_ranks(_timed_calls(p_rs, stream, n))
        one.close()
        tail_ag = max_over_ranks(traced_tail(comm, ag, dev))
        tail_rs = max_over_ranks(traced_tail(comm, rs, dev))
    else:
        plain_ag, plain_rs, tail_ag, tail_rs = ag_ms, rs_ms, 0.0, 0.0
    exposed = {"ag_us": 1e3 * (ag_ms - plain_ag), "rs_us": 1e3 * (rs_ms - plain_rs),
               "block_us": 1e3 * (ag_ms + rs_ms - plain_ag - plain_rs),
               "definition": "t(fused op) - t(plain per-rank GEMM of the same shapes), device events, max over ranks"}

    # ---- e2e through the public API with pinned host buffers (copies timed).
    # Every step copies its input from pinned host memory and its result back; the copies
    # run on their own streams (copy engines), double-buffered so step i+1's H2D and step
    # i-1's D2H overlap step i's kernels.
    nbuf = 2
    x_host = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for _ in range(nbuf)]
    y_host = [torch.empty(y.shape, dtype=y.dtype, pin_memory=True) for _ in range(nbuf)]
    for hbuf in x_host:
        hbuf.copy_(x.cpu())
    x_dev = [torch.empty_like(x) for _ in range(nbuf)]
    y_dev = [torch.empty_like(y) for _ in range(nbuf)]
    e2e_ms = max_over_ranks(e2e_pipeline(torch, n, x_host, y_host, x_dev, y_dev,
                                          lambda xin, yout: (ag(xin), rs(yout)), stream, dev, barrier))
    e2e_value = flops_step / (e2e_ms * 1e-3) / 1e12
    h2d = x_host[0].numel() * x_host[0].element_size() * world
    d2h = y_host[0].numel() * y_host[0].element_size() * world

    # ---- non-overlapped baseline in the same run: cuBLAS (+ NCCL all-gather / reduce-scatter
    # for T > 1), the reference's "baseline" strategy (experiment.cpp:789-836, fabric.cpp:132-181)
    base = None
    try:
        xg = torch.empty((1, SEQ, D_MODEL), device=dev, dtype=torch.bfloat16)
        yfull = torch.empty((1, SEQ, D_MODEL), device=dev, dtype=torch.bfloat16)
        bev = []

        def base_step(rec=False):
            e = _events(1, 4)[0] if rec else None
            if e:
                e[0].record(stream)
            if T > 1:
                dist.all_gather_into_tensor(xg, x)
            else:
                xg.copy_(x)
            if e:
                e[1].record(stream)
            gt = torch.matmul(xg.view(SEQ, D_MODEL), w_gate)
            up = torch.matmul(xg.view(SEQ, D_MODEL), w_up)
            a = torch.nn.functional.silu(gt) * up
            torch.matmul(a, w_dn, out=yfull.view(SEQ, D_MODEL))
            if e:
                e[2].record(stream)
            if T > 1:
                dist.reduce_scatter_tensor(y, yfull)
            if e:
                e[3].record(stream)
                bev.append(e)
        for _ in range(max(2, args.warmup)):
            base_step()
        torch.cuda.synchronize(dev)
        barrier()
        for _ in range(n):
            base_step(True)
        torch.cuda.synchronize(dev)
        base_ms = max_over_ranks(bev[0][0].elapsed_time(bev[-1][3]) / n)
        comm_ms = max_over_ranks(sum(e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3]) for e in bev) / n)
        base = {"ms_per_step": base_ms, "tflops": flops_step / (base_ms * 1e-3) / 1e12,
                "collectives_ms": comm_ms if T > 1 else 0.0, "speedup_ours": base_ms / ms_step,
                "what": ("NCCL all_gather_into_tensor + cuBLAS gate/up + SwiGLU + cuBLAS down + NCCL "
                         "reduce_scatter_tensor, non-overlapped" if T > 1 else "cuBLAS gate/up + SwiGLU + cuBLAS down")}
    except Exception as exc:  # baseline is informative only
        print(f"[bench] baseline failed: {exc}", file=sys.stderr)

    # ---- CPU reference sample (rank 0 at N = 1). It runs before the per-GPU blocks below, so
    # the GPU idles ~10 s after the sustained bench load and those blocks start cool.
    cpu = None
    if world == 1 and not args.no_cpu:
        nproc = os.cpu_count() or 1
        cbs = cpu_reference_sample(max(1, min(8, nproc)), 8)
        cb = cbs[0] if cbs else None
        if cb:
            cpu = {"value": cb["tflops"], "unit": "TFLOP/s", "cores": cb["ranks"], "kind": "reference",
                   "sample": f"{cb['tokens']} tokens of the block ({cb['ranks']} simulated TP ranks, "
                             f"one thread each), {cb['seconds']:.1f} s of reference CPU work, host nproc={nproc}"}

    # ---- one GPU of a TP=8 group at full scale (virtual peers)
    virt = None
    if world == 1 and args.emulate_tp > 1:
        virt = virtual_block(args, dev, stream, args.emulate_tp)
    others = None
    if world == 1 and args.emulate_tp > 1 and not args.no_other_configs:
        others = other_configs_block(dev, stream)

    comm.close()
    if rank != 0:
        return
    pk = peaks()
    ag_flops = 2.0 * SEQ * D_MODEL * (2 * F_l)  # per rank per launch
    achieved = ag_flops / (ag_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(f"ag_gemm_tp{T}")
    out = {
        "metric": METRIC,
        "value": value,
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": n,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded randn, random-init weights of the Llama-3-8B MLP shapes)",
        "config": {"workload": WORKLOAD, "tp": T, "seq_len": SEQ, "global_batch": 1, "d_model": D_MODEL,
                   "ffn": FFN, "parallelism": f"tp{T}-sp" if T > 1 else "tp1 (degenerate: plain GEMMs)",
                   "rs_schedule": "ring", "rs_wire": "bf16",
                   "l2": "no flush: per-step working set ~1.0 GB (weights 352 MB + hidden 470 MB) > 126 MB L2"},
        "gpu_launches": 2 * n,
        "ops": {
            "ag_gemm_swiglu": {"ms": ag_ms, "tflops": 2.0 * SEQ * D_MODEL * 2 * FFN / (ag_ms * 1e-3) / 1e12,
                               "plain_gemm_ms": plain_ag, "fused_over_plain": ag_ms / plain_ag,
                               "tail_us": tail_ag,
                               "note": "AG-GEMM gate||up with SwiGLU fused in the epilogue"},
            "gemm_rs": {"ms": rs_ms, "tflops": 2.0 * SEQ * FFN * D_MODEL / (rs_ms * 1e-3) / 1e12,
                        "plain_gemm_ms": plain_rs, "fused_over_plain": rs_ms / plain_rs, "tail_us": tail_rs},
            "exposed_comm_us": exposed,
            "no_tail": tail_ag == 0.0 and tail_rs == 0.0,
        },
        "roofline": {"kernel": "tpf_fused_kernel (AG-GEMM gate||up + fused SwiGLU)", "bound": "tensor",
                     "achieved": achieved, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                     "frac": achieved / pk["bf16_tflops"], "traffic": traffic,
                     "peak_src": f"{pk['src']} burst; frac vs sustained {pk['bf16_tflops_sustained']}: "
                                 f"{achieved / pk['bf16_tflops_sustained']:.3f}",
                     "flops_per_launch": ag_flops,
                     "frac_vs_spec_dense_2250": achieved / 2250.0},
        "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms, "gpu_launches": 2 * n,
                "how": "C-ABI calls; pinned host x -> device and y -> host every step, copies on "
                       "separate streams double-buffered against the kernels"},
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    if base:
        out["baseline_cublas_nccl"] = base
    if virt:
        out["virtual_per_gpu"] = virt
    if others:
        out["other_configs"] = others
    print(json.dumps(out))


def other_configs_block(dev, stream):
    """The other BASELINE configurations, measured in the same run (informational; the headline
    is cfg2): one GPU of a TP = 8 group (virtual peers) on the cfg3 attention projections, one
    GPU of the 8-rank DP group of cfg4, and the cfg5 UP layer (all 8 ranks on this GPU, each on
    148/8 SMs). Fused vs plain per-rank GEMM; medians of 3 alternating rounds."""
    import statistics

    import torch

    import paper_2604_24013_b200 as tpf
    pk = peaks()["bf16_tflops"] * 1e12
    one = tpf.Communicator.create(0, 1, 0)
    g = torch.Generator(device=dev).manual_seed(21)
    res = {}

    def pair(fused, plain, rounds=3):
        for _ in range(2):
            fused(); plain()
        f, q = [], []
        for _ in range(rounds):
            f.append(_timed_calls(fused, stream, 10))
            q.append(_timed_calls(plain, stream, 10))
        return statistics.median(f), statistics.median(q)

    def row(fms, pms, flops, wire):
        roof = max(flops / pk, wire / 900e9) * 1e3
        return {"fused_ms": fms, "plain_gemm_ms": pms, "fused_over_plain": fms / pms,
                "exposed_us": 1e3 * (fms - pms), "tflops": flops / (fms * 1e-3) / 1e12,
                "t_roof_ms": roof, "frac_of_t_roof": roof / fms}

    T, S, K = 8, 16384, 8192
    x = torch.randn((1, S // T, K), device=dev, generator=g).to(torch.bfloat16)
    xg = torch.randn((1, S, K), device=dev, generator=g).to(torch.bfloat16)
    wq = (torch.randn((K, 10240 // T), device=dev, generator=g) / 90).to(torch.bfloat16)
    yq = torch.empty((1, S, 10240 // T), device=dev, dtype=torch.bfloat16)
    xo = torch.randn((1, S, K // T), device=dev, generator=g).to(torch.bfloat16)
    wo = (torch.randn((K // T, K), device=dev, generator=g) / 90).to(torch.bfloat16)
    yo = torch.empty((1, S // T, K), device=dev, dtype=torch.bfloat16)
    yog = torch.empty((1, S, K), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, S, K, 10240 // T),
                                                 tpf.sym_bytes_rs(T, 1, S, K // T, K, 1, tpf.BF16)))
    fq, pq = pair(lambda: comm.ag_gemm(x, wq, yq, stream=stream), lambda: one.ag_gemm(xg, wq, yq, stream=stream))
    fo, po = pair(lambda: comm.gemm_rs(xo, wo, yo, kind=tpf.RING, wire=tpf.BF16, stream=stream),
                  lambda: one.gemm_rs(xo, wo, yog, stream=stream))
    comm.sync(stream)
    comm.close()
    moved = (T - 1) / T * S * 2
    res["cfg3_tp8_per_gpu"] = {"qkv_ag_gemm": row(fq, pq, 2.0 * S * K * 10240 / T, moved * K),
                               "out_proj_gemm_rs_bf16_wire": row(fo, po, 2.0 * S * K * K / T, moved * K)}
    del x, xg, wq, yq, xo, wo, yo, yog
    M, K4, N4 = 4096, 2048, 8192
    X = torch.randn((M, K4), device=dev, generator=g).to(torch.bfloat16)
    dY = (torch.randn((M, N4), device=dev, generator=g) / 64).to(torch.bfloat16)
    dW = torch.empty((K4 // T, N4), device=dev, dtype=torch.bfloat16)
    dWf = torch.empty((K4, N4), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.virtual_group(T, tpf.sym_bytes_rs(T, 1, K4, M, N4, 1, tpf.BF16))
    fd, pd = pair(lambda: comm.dp_grad_rs(X, dY, dW, kind=tpf.RING, wire=tpf.BF16, stream=stream),
                  lambda: one.dp_grad_rs(X, dY, dWf, stream=stream))
    comm.sync(stream)
    comm.close()
    res["cfg4_dp8_per_gpu"] = {"grad_rs_bf16_wire": row(fd, pd, 2.0 * M * K4 * N4, (T - 1) / T * K4 * N4 * 2),
                               "shape": "4096 tokens / rank, 2048 x 8192 weight"}
    del X, dY, dW, dWf
    heads, S5 = 4, 32768
    q, k, v = (torch.randn((T, heads, S5, 128), device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
    o = torch.empty((T, 1, S5 // T, T * heads * 128), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ulysses(T, 1, T * heads, S5, 128))
    up = lambda: comm.attention_a2a(q, k, v, o, 1, heads, stream=stream)  # noqa: E731
    up()
    ms = statistics.median(_timed_calls(up, stream, 2) for _ in range(3))
    comm.sync(stream)
    comm.close()
    res["cfg5_up_attention_local_group"] = {
        "ms": ms, "tflops": 4.0 * T * heads * S5 * S5 * 128 / (ms * 1e-3) / 1e12,
        "note": "fuse_all_to_all_attention, T = 8 ranks on this GPU (each on 148/8 SMs), 4 heads x 128 per "
                "rank, S = 32768, non-causal; the output all-to-all is fused in the epilogue"}
    one.close()
    return res


def virtual_block(args, dev, stream, T):
    """One GPU of a real TP=T group at full scale: rank 0 with virtual peers (a self-ring: the
    peers alias this rank's heap, so every send fills the slot this rank reads one step later
    and the ring's step-to-step dependencies are real, with zero link latency) runs the cfg2
    block's per-rank AG-GEMM + SwiGLU and GEMM-RS with the whole protocol, against the plain
    per-rank GEMMs of the same shapes (acceptance C6: fused / plain), and a traced call of each
    for the measured tail. NVLink latency is the part it cannot show."""
    import statistics

    import torch

    import paper_2604_24013_b200 as tpf
    S_l, F_l = SEQ // T, FFN // T
    g = torch.Generator(device=dev).manual_seed(11)
    x = torch.randn((1, S_l, D_MODEL), device=dev, generator=g).to(torch.bfloat16)
    xg = torch.randn((1, SEQ, D_MODEL), device=dev, generator=g).to(torch.bfloat16)
    w_gu = (torch.randn((D_MODEL, 2 * F_l), device=dev, generator=g) / 64).to(torch.bfloat16)
    w_dn = (torch.randn((F_l, D_MODEL), device=dev, generator=g) / 120).to(torch.bfloat16)
    act = torch.empty((1, SEQ, F_l), device=dev, dtype=torch.bfloat16)
    y = torch.empty((1, S_l, D_MODEL), device=dev, dtype=torch.bfloat16)
    y32 = torch.empty((1, S_l, D_MODEL), device=dev, dtype=torch.float32)
    yg = torch.empty((1, SEQ, D_MODEL), device=dev, dtype=torch.bfloat16)
    comm = tpf.Communicator.virtual_group(T, max(tpf.sym_bytes_ag(T, 1, SEQ, D_MODEL, 2 * F_l, 1),
                                                 tpf.sym_bytes_rs(T, 1, SEQ, F_l, D_MODEL, 1, tpf.F32)))
    one = tpf.Communicator.create(0, 1, 0)

    ag = lambda: comm.ag_gemm(x, w_gu, act, act=tpf.ACT_SWIGLU, stream=stream)  # noqa: E731
    rs = lambda: comm.gemm_rs(act, w_dn, y, kind=tpf.RING, wire=tpf.BF16, stream=stream)  # noqa: E731
    rs32 = lambda: comm.gemm_rs(act, w_dn, y32, kind=tpf.RING, wire=tpf.F32, stream=stream)  # noqa: E731
    p_ag = lambda: one.ag_gemm(xg, w_gu, act, act=tpf.ACT_SWIGLU, stream=stream)  # noqa: E731
    p_rs = lambda: one.gemm_rs(act, w_dn, yg, stream=stream)  # noqa: E731
    for _ in range(3):
        ag(); rs(); rs32(); p_ag(); p_rs()
    res = {"ag": [], "rs": [], "rs32": [], "p_ag": [], "p_rs": []}
    fns = {"ag": ag, "rs": rs, "rs32": rs32, "p_ag": p_ag, "p_rs": p_rs}
    for _ in range(5):  # rounds alternate fused and plain, so both see the same power state
        for k, fn in fns.items():
            res[k].append(_timed_calls(fn, stream, 20))
    comm.sync(stream)
    tail_ag = traced_tail(comm, ag, dev)
    tail_rs = traced_tail(comm, rs, dev)
    comm.close()
    one.close()
    m = {k: statistics.median(v) for k, v in res.items()}
    fl_ag, fl_rs = 2.0 * SEQ * D_MODEL * 2 * F_l, 2.0 * SEQ * F_l * D_MODEL
    # SURVEY 8(d) roofline: max(FLOPs at the measured bf16 burst peak, NVLink bytes at 900 GB/s)
    pk = peaks()["bf16_tflops"] * 1e12
    rows_moved = (T - 1) / T * SEQ
    t_roof_ag = max(fl_ag / pk, rows_moved * D_MODEL * 2 / 900e9) * 1e3
    t_roof_rs = max(fl_rs / pk, rows_moved * D_MODEL * 2 / 900e9) * 1e3
    t_roof_rs32 = max(fl_rs / pk, rows_moved * D_MODEL * 4 / 900e9) * 1e3
    # the same with the pool's measured peer-copy rate, 770 GB/s per direction
    # (/opt/skills/guides/B200_PROFILING.md): the RS bf16 wire is then link-bound at TP = 8
    m_ag = max(fl_ag / pk, rows_moved * D_MODEL * 2 / 770e9) * 1e3
    m_rs = max(fl_rs / pk, rows_moved * D_MODEL * 2 / 770e9) * 1e3
    m_rs32 = max(fl_rs / pk, rows_moved * D_MODEL * 4 / 770e9) * 1e3
    return {"tp": T, "note": "one GPU of a TP group at full scale: rank 0 with virtual peers (self-ring: "
                             "peers alias the own heap, sends fill the slot read one step later, zero link "
                             "latency); medians of 5 rounds of 20 back-to-back calls per op; plain = the T = 1 "
                             "kernel on the same per-rank shapes",
            "ag_gemm_ms": m["ag"], "gemm_rs_ms": m["rs"], "gemm_rs_f32_wire_ms": m["rs32"],
            "plain_ag_gemm_ms": m["p_ag"], "plain_gemm_rs_ms": m["p_rs"],
            "fused_over_plain": {"ag": m["ag"] / m["p_ag"], "rs": m["rs"] / m["p_rs"]},
            "exposed_comm_us": {"ag": 1e3 * (m["ag"] - m["p_ag"]), "rs": 1e3 * (m["rs"] - m["p_rs"])},
            "tail_us": {"ag": tail_ag, "rs": tail_rs},
            "ag_tflops_per_gpu": fl_ag / (m["ag"] * 1e-3) / 1e12, "rs_tflops_per_gpu": fl_rs / (m["rs"] * 1e-3) / 1e12,
            "t_roof_ms": {"ag": t_roof_ag, "rs": t_roof_rs, "rs_f32_wire": t_roof_rs32,
                          "how": "max(FLOPs at the measured bf16 burst peak, NVLink bytes at 900 GB/s) (north_star)"},
            "frac_of_t_roof": {"ag": t_roof_ag / m["ag"], "rs": t_roof_rs / m["rs"],
                               "rs_f32_wire": t_roof_rs32 / m["rs32"]},
            "t_roof_ms_link770": {"ag": m_ag, "rs": m_rs, "rs_f32_wire": m_rs32,
                                  "how": "NVLink at the measured 770 GB/s peer copy (profiling guide)"},
            "frac_of_t_roof_link770": {"ag": m_ag / m["ag"], "rs": m_rs / m["rs"], "rs_f32_wire": m_rs32 / m["rs32"]}}


# ------------------------------------------------------------- launch / dry run
def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args) -> int:
    """`bench.py --gpus N` without a torchrun environment: launch N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 and return the group's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args, rank, world):
    """--dry-run: the multi-rank harness without GPUs (gloo): rendezvous, barrier, max-over-ranks
    reduction and the one JSON line from rank 0. Used by the CPU test of the launcher."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "ranks_seen": int(t.item()),
                          "steps": args.steps, "warmup": args.warmup, "impl": args.impl}))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--emulate-tp", type=int, default=8, help="per-GPU TP group model at N=1 (0 = off)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU reference sample")
    ap.add_argument("--no-other-configs", action="store_true", help="skip the cfg3 / cfg4 / cfg5 block (N=1)")
    ap.add_argument("--dry-run", action="store_true", help="launcher / rank plumbing only (gloo, no GPU)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU", file=sys.stderr)
        sys.exit(2)
    if args.dry_run:
        run_dry(args, rank, world)
        return
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
