"""Three-strategy bench in the reference's CSV wire format.

Mirrors ``run_bench`` / ``run_bench_collect`` (reference proj/src/experiment.cpp:789-860):
the same layers (mlp, attention, ulysses, rs, ag), the same three
strategies, the same warm-up agreement check ("bench strategies disagree on layer
output"), round-robin interleaved repetitions, ``chunk_compute_ms`` from one
partial-output compute, and the byte-identical header ``BENCH_CSV_HEADER``
(experiment.cpp:838-840) with the row format of experiment.cpp:846-855.

What runs on the B200, per strategy (``make_bench_setup``, experiment.cpp:567-753):
  baseline      compute everything (cuBLAS / SDPA), THEN the collective (not overlapped)
  data-slicing  per-destination-slice compute in natural order, each slice shipped to its
                owner on a side stream as soon as it is ready, settled at the end
                (``sliced_row_parallel``, experiment.cpp:533-558)
  fused         this library's fused kernels (ag_gemm / gemm_rs / query_split_attention /
                attention_a2a) with the configured schedule and granularity

The group is the single-GPU local group (all tp_size ranks on one B200, as in every
GPU test here): the fused arm moves its wire bytes through the symmetric heap, and the
baseline / data-slicing arms move the same bytes with device copies and reductions on
that GPU. On one GPU those copies run at HBM speed, not NVLink speed, so this emulation
favours the non-fused arms. Times come from CUDA events, in ms per layer call.

    python -m paper_2604_24013_b200.benchcsv --layer mlp --tp_size 4 --batch 1 --seq 8192 \
        --d_model 4096 --reps 10 > bench.csv
"""
from __future__ import annotations

import argparse
import dataclasses
import math
import sys
from typing import Callable, Dict, List

import paper_2604_24013_b200 as tpf

BENCH_CSV_HEADER = ("strategy,layer,tp_size,batch,seq,d_model,heads,granularity,schedule,seed,"
                    "delay_ms,reps,chunk_compute_ms,mean_ms,latency_reduction_pct")
STRATEGIES = ("baseline", "data-slicing", "fused")
LAYERS = ("mlp", "attention", "ulysses", "rs", "ag")
SCHEDULES = {"ring": tpf.RING, "pairwise": tpf.PAIRWISE, "circular-slices": tpf.CIRCULAR}


@dataclasses.dataclass
class BenchConfig:
    """ExperimentConfig (experiment.hpp:28-42): same fields, same defaults."""
    tp_size: int = 4
    batch: int = 2
    seq: int = 64
    d_model: int = 32
    heads: int = 4
    granularity: int = 1
    schedule: str = "ring"
    layer: str = "mlp"
    seed: int = 0
    delay_ms: float = 0.0
    reps: int = 10

    def validate(self) -> None:
        """ExperimentConfig::validate (experiment.cpp:50-93) plus the GPU path's limits."""
        t = self.tp_size
        if t < 1:
            raise ValueError("tp_size must be >= 1")
        if self.batch < 1 or self.seq < 1 or self.d_model < 1 or self.heads < 1:
            raise ValueError("batch, seq, d_model and heads must be >= 1")
        if self.granularity < 1:
            raise ValueError("granularity must be >= 1")
        if self.reps < 1:
            raise ValueError("reps must be >= 1")
        if self.seq % (t * self.granularity):
            raise ValueError(f"seq ({self.seq}) must be divisible by tp_size*granularity ({t * self.granularity})")
        if self.delay_ms != 0.0:
            raise ValueError("delay_ms is a CPU-fabric knob; the GPU bench measures real transfers (use 0)")
        if self.layer not in LAYERS:
            raise ValueError(f"unknown layer '{self.layer}'")
        if self.schedule not in SCHEDULES:
            raise ValueError(f"unknown schedule '{self.schedule}'")
        if self.schedule == "pairwise" and t > 1 and t % 2:
            raise ValueError("pairwise schedule needs an even tp_size")
        if self.layer in ("attention", "ulysses"):
            if self.heads % t:
                raise ValueError(f"heads ({self.heads}) must be divisible by tp_size ({t})")
            if self.d_model % self.heads:
                raise ValueError(f"d_model ({self.d_model}) must be divisible by heads ({self.heads})")
            if self.granularity != 1:
                raise ValueError("attention layers support granularity = 1 only")
            if self.d_model // self.heads != 128:
                raise ValueError("the fused attention kernel needs head_dim = d_model / heads = 128")
        if self.layer == "mlp" and self.d_model % t:
            raise ValueError(f"d_model ({self.d_model}) must be divisible by tp_size ({t})")
        if self.layer in ("mlp", "rs") and self.granularity > 1 and self.schedule != "ring":
            raise ValueError("fuse_reduce_scatter: granularity > 1 is supported for the ring schedule only")
        if self.layer in ("mlp", "attention", "rs", "ag") and (self.d_model * 2) % 16:
            raise ValueError("d_model rows must be 16-byte aligned in bf16 (d_model % 8 == 0)")


@dataclasses.dataclass
class BenchMeasurement:
    strategy: str
    mean_ms: float
    latency_reduction_pct: float = 0.0


@dataclasses.dataclass
class BenchResult:
    chunk_compute_ms: float
    measurements: List[BenchMeasurement]


def format_row(cfg: BenchConfig, chunk_compute_ms: float, m: BenchMeasurement) -> str:
    """One CSV row, printf format of experiment.cpp:849 ("%.10g" for the doubles)."""
    g = lambda v: "%.10g" % v  # noqa: E731
    return ",".join([m.strategy, cfg.layer, str(cfg.tp_size), str(cfg.batch), str(cfg.seq), str(cfg.d_model),
                     str(cfg.heads), str(cfg.granularity), cfg.schedule, str(cfg.seed), g(cfg.delay_ms),
                     str(cfg.reps), g(chunk_compute_ms), g(m.mean_ms), g(m.latency_reduction_pct)])


def format_csv(cfg: BenchConfig, result: BenchResult) -> str:
    lines = [BENCH_CSV_HEADER] + [format_row(cfg, result.chunk_compute_ms, m) for m in result.measurements]
    return "\n".join(lines) + "\n"


def latency_reductions(measurements: List[BenchMeasurement]) -> None:
    """Against the first (baseline) strategy, experiment.cpp:832-835."""
    base = measurements[0].mean_ms
    for m in measurements:
        m.latency_reduction_pct = (base - m.mean_ms) / base * 100.0 if base > 0 else 0.0


# ------------------------------------------------------------------ GPU setup
def _randint(torch, shape, lo, hi, seed, dev):
    g = torch.Generator(device=dev).manual_seed(seed)
    return torch.randint(lo, hi, shape, generator=g, device=dev, dtype=torch.int32).to(torch.bfloat16)


class _Setup:
    """body[strategy]() runs one layer call for all ranks; out() returns the per-rank outputs
    (rank-stacked) of the last call; chunk() is one partial-output compute for all ranks."""

    def __init__(self):
        self.body: Dict[str, Callable[[], None]] = {}
        self.out: Dict[str, Callable[[], object]] = {}
        self.chunk: Callable[[], None] = lambda: None
        self.tol = 1e-6
        self.comm = None


def _sliced_settle(torch, T, side, make_slice, inbox, own_out):
    """Data-slicing (experiment.cpp:533-558) for all ranks: slice s computed for every rank
    (batched), shipped to owner s on the side stream as soon as it is ready; the owner then
    accumulates its T contributions (own slice included) in source order."""
    cur = torch.cuda.current_stream()
    for s in range(T):
        y = make_slice(s)  # (T_src, ...) contribution of every source rank for owner s
        ev = torch.cuda.Event()
        ev.record(cur)
        side.wait_event(ev)
        with torch.cuda.stream(side):
            inbox[s].copy_(y)
            y.record_stream(side)
    done = torch.cuda.Event()
    done.record(side)
    cur.wait_event(done)
    own_out(inbox)


def make_setup(cfg: BenchConfig):
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    T, B, S, D, seed = cfg.tp_size, cfg.batch, cfg.seq, cfg.d_model, cfg.seed
    kind = SCHEDULES[cfg.schedule]
    sl = S // T
    st = _Setup()
    side = torch.cuda.Stream(device=dev)

    if cfg.layer in ("mlp", "rs"):
        if cfg.layer == "mlp":
            # experiment.cpp:574-610: x (B,S,D) in [0,3), up (D,2D) / down (2D,D) in [-2,2];
            # the up half (all-gather + matmul + tanh) is conventional in every strategy.
            H = 2 * D
            x = _randint(torch, (B, S, D), 0, 3, seed * 1000 + 0, dev)
            up = _randint(torch, (D, H), -2, 3, seed * 1000 + 1, dev).view(D, T, H // T).permute(1, 0, 2).contiguous()
            down = _randint(torch, (H, D), -2, 3, seed * 1000 + 2, dev).view(T, H // T, D).contiguous()
            act = torch.empty((T, B, S, H // T), device=dev, dtype=torch.bfloat16)

            def up_half():
                torch.bmm(x.view(1, B * S, D).expand(T, B * S, D), up, out=act.view(T, B * S, H // T))
                act.tanh_()
            K_loc, xin, w = H // T, act, down
            st.tol = 1e-5
        else:
            # experiment.cpp:693-716: each rank's (B,S,D) input in [0,3), identity compute
            up_half = lambda: None  # noqa: E731
            K_loc = D
            xin = torch.stack([_randint(torch, (B, S, D), 0, 3, seed * 1000 + q, dev)[0:B] for q in range(T)])
            w = torch.eye(D, device=dev, dtype=torch.bfloat16).expand(T, D, D).contiguous()
        N = D
        part = torch.empty((T, B, S, N), device=dev, dtype=torch.float32)
        outs = {s: torch.empty((T, B, sl, N), device=dev, dtype=torch.float32) for s in STRATEGIES}
        inbox = [torch.empty((T, B, sl, N), device=dev, dtype=torch.float32) for _ in range(T)]
        comm = tpf.Communicator.local_group(T, tpf.sym_bytes_rs(T, B, S, K_loc, N, cfg.granularity, tpf.F32))
        st.comm = comm

        def baseline():
            up_half()
            # every rank's full fp32 partial output, then the reduce-scatter (not overlapped)
            part.view(T, B * S, N).copy_(torch.bmm(xin.view(T, B * S, K_loc), w, out_dtype=torch.float32))
            outs["baseline"].copy_(part.view(T, B, T, sl, N).sum(0).permute(1, 0, 2, 3))

        def slice_gemm(s):
            a = xin[:, :, s * sl:(s + 1) * sl].reshape(T, B * sl, K_loc)
            return torch.bmm(a, w, out_dtype=torch.float32).view(T, B, sl, N)

        def sliced():
            up_half()
            make_slice = slice_gemm

            def settle(ib):
                torch.sum(torch.stack(ib), 1, out=outs["data-slicing"])

            _sliced_settle(torch, T, side, make_slice, inbox, settle)

        def fused():
            up_half()
            comm.gemm_rs(xin, w, outs["fused"], kind=kind, m=cfg.granularity, wire=tpf.F32)

        st.body = {"baseline": baseline, "data-slicing": sliced, "fused": fused}
        st.chunk = lambda: slice_gemm(0)
        st.out = {s: (lambda s=s: outs[s]) for s in STRATEGIES}
        return st

    if cfg.layer == "ag":
        # experiment.cpp:718-739: each rank's (B,S/T,D) slice in [0,3); baseline and
        # data-slicing are both the plain all-gather. The fused path's partial compute is a
        # GEMM, so f = matmul(I) here, and the two conventional arms apply the same f after
        # their all-gather so that all three compute the same function.
        xin = torch.stack([_randint(torch, (B, sl, D), 0, 3, seed * 1000 + q, dev) for q in range(T)])
        eye = torch.eye(D, device=dev, dtype=torch.bfloat16).expand(T, D, D).contiguous()
        outs = {s: torch.empty((T, B, S, D), device=dev, dtype=torch.float32) for s in STRATEGIES}
        comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ag(T, B, S, D, D, cfg.granularity))
        st.comm = comm

        gathered = torch.empty((T, B * S, D), device=dev, dtype=torch.bfloat16)

        def gather(name):
            def run():
                gathered.view(T, B, S, D).copy_(xin.permute(1, 0, 2, 3).reshape(B, S, D).unsqueeze(0))
                outs[name].view(T, B * S, D).copy_(torch.bmm(gathered, eye, out_dtype=torch.float32))
            return run

        st.body = {"baseline": gather("baseline"), "data-slicing": gather("data-slicing"),
                   "fused": lambda: comm.ag_gemm(xin, eye, outs["fused"], m=cfg.granularity)}
        st.chunk = lambda: xin.clone()
        st.out = {s: (lambda s=s: outs[s]) for s in STRATEGIES}
        return st

    # attention / ulysses: build_attention_data analogue -- per rank q/k/v for its head group
    h = cfg.heads // T
    Dh = 128
    g = torch.Generator(device=dev).manual_seed(seed)
    q, k, v = ((torch.rand((T, B * h, S, Dh), generator=g, device=dev) * 2 - 1).to(torch.bfloat16)
               for _ in range(3))
    sdpa = torch.nn.functional.scaled_dot_product_attention
    st.tol = 2e-2

    def merged(ctx, rows):  # (T, B*h, rows, Dh) -> (T, B, rows, h*Dh)
        return ctx.view(T, B, h, rows, Dh).permute(0, 1, 3, 2, 4).reshape(T, B, rows, h * Dh)

    if cfg.layer == "attention":
        w_o = ((torch.rand((T, h * Dh, D), generator=g, device=dev) * 2 - 1) / 16).to(torch.bfloat16)
        outs = {s: torch.empty((T, B, sl, D), device=dev, dtype=torch.float32) for s in STRATEGIES}
        inbox = [torch.empty((T, B, sl, D), device=dev, dtype=torch.float32) for _ in range(T)]
        comm = tpf.Communicator.local_group(T, tpf.sym_bytes_rs(T, B, S, h * Dh, D, 1, tpf.F32) + (1 << 22))
        st.comm = comm

        def baseline():
            ctx = merged(sdpa(q, k, v), S)
            part = torch.matmul(ctx, w_o.unsqueeze(1)).float()
            outs["baseline"].copy_(part.view(T, B, T, sl, D).sum(0).permute(1, 0, 2, 3))

        def sliced():
            def make_slice(s):
                ctx = merged(sdpa(q[:, :, s * sl:(s + 1) * sl], k, v), sl)
                return torch.matmul(ctx, w_o.unsqueeze(1)).float()

            _sliced_settle(torch, T, side, make_slice, inbox,
                           lambda ib: torch.sum(torch.stack(ib), 1, out=outs["data-slicing"]))

        st.body = {"baseline": baseline, "data-slicing": sliced,
                   "fused": lambda: comm.query_split_attention(q, k, v, w_o, outs["fused"], B, h, kind=kind)}
        st.chunk = lambda: torch.matmul(merged(sdpa(q[:, :, :sl], k, v), sl), w_o.unsqueeze(1))
    else:  # ulysses, experiment.cpp:644-691
        F = T * h * Dh
        outs = {s: torch.empty((T, B, sl, F), device=dev, dtype=torch.bfloat16) for s in STRATEGIES}
        comm = tpf.Communicator.local_group(T, tpf.sym_bytes_ulysses(T, B, cfg.heads, S, Dh))
        st.comm = comm

        def a2a_into(out, ctx_slices):
            # owner r's feature block src holds source src's merged context for slice r
            for src in range(T):
                out[:, :, :, src * h * Dh:(src + 1) * h * Dh].copy_(ctx_slices[src])

        def baseline():
            ctx = merged(sdpa(q, k, v), S)  # (T_src, B, S, h*Dh)
            a2a_into(outs["baseline"], [ctx[src].view(B, T, sl, h * Dh).permute(1, 0, 2, 3) for src in range(T)])

        def sliced():
            cur = torch.cuda.current_stream()
            for s in range(T):
                ctx = merged(sdpa(q[:, :, s * sl:(s + 1) * sl], k, v), sl)  # (T_src, B, sl, h*Dh)
                ev = torch.cuda.Event()
                ev.record(cur)
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    outs["data-slicing"][s].copy_(ctx.permute(1, 2, 0, 3).reshape(B, sl, F))
                    ctx.record_stream(side)
            done = torch.cuda.Event()
            done.record(side)
            cur.wait_event(done)

        st.body = {"baseline": baseline, "data-slicing": sliced,
                   "fused": lambda: comm.attention_a2a(q, k, v, outs["fused"], B, h)}
        st.chunk = lambda: merged(sdpa(q[:, :, :sl], k, v), sl)
    st.out = {s: (lambda s=s: outs[s]) for s in STRATEGIES}
    return st


def _rel_deviation(a, b) -> float:
    a, b = a.double(), b.double()
    scale = b.abs().max().item()
    return (a - b).abs().max().item() / (scale if scale > 0 else 1.0)


def _time_ms(torch, fn) -> float:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def measure_chunk_compute_ms(cfg: BenchConfig, st: _Setup = None) -> float:
    """experiment.cpp:757-787: one partial-output compute for every rank at once (the
    reference runs tp_size copies concurrently); median of 5 after one warm-up."""
    import torch
    st = st or make_setup(cfg)
    st.chunk()
    samples = sorted(_time_ms(torch, st.chunk) for _ in range(5))
    return samples[len(samples) // 2]


def run_bench_collect(cfg: BenchConfig) -> BenchResult:
    """run_bench_collect (experiment.cpp:789-836) on the B200."""
    import torch
    cfg.validate()
    st = make_setup(cfg)
    try:
        chunk_ms = measure_chunk_compute_ms(cfg, st)
        # warm-up round, discarded; the strategies must agree on the math they time
        base = None
        for s in STRATEGIES:
            st.body[s]()
            st.comm.sync()
            out = st.out[s]()
            if base is None:
                base = out.clone()
            elif not torch.isfinite(out).all() or _rel_deviation(out, base) > st.tol:
                raise tpf.LogicError("bench strategies disagree on layer output")
        totals = dict.fromkeys(STRATEGIES, 0.0)
        for _ in range(cfg.reps):  # round-robin so drift lands on all strategies equally
            for s in STRATEGIES:
                totals[s] += _time_ms(torch, st.body[s])
        st.comm.sync()
    finally:
        st.comm.close()
    ms = [BenchMeasurement(s, totals[s] / cfg.reps) for s in STRATEGIES]
    latency_reductions(ms)
    return BenchResult(chunk_ms, ms)


def run_bench(cfg: BenchConfig, out=sys.stdout) -> int:
    """run_bench (experiment.cpp:842-860): header plus one row per strategy."""
    out.write(format_csv(cfg, run_bench_collect(cfg)))
    return 0


def parse_args(argv=None) -> BenchConfig:
    p = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    d = BenchConfig()
    for f in dataclasses.fields(BenchConfig):
        p.add_argument("--" + f.name, type=type(getattr(d, f.name)), default=getattr(d, f.name))
    a = p.parse_args(argv)
    cfg = BenchConfig(**{f.name: getattr(a, f.name) for f in dataclasses.fields(BenchConfig)})
    cfg.validate()
    return cfg


if __name__ == "__main__":
    sys.exit(run_bench(parse_args()))
