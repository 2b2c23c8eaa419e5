"""Bench CSV wire format: the GPU three-strategy bench writes the
reference's kBenchCsvHeader schema (experiment.cpp:838-860), checked against the
reference's own run_bench output; the GPU run itself is a -m gpu test."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_24013_b200 import benchcsv as bc  # noqa: E402

from oracle_lib import Reference, have_reference  # noqa: E402

# experiment.cpp:838-840, verbatim
REF_HEADER = ("strategy,layer,tp_size,batch,seq,d_model,heads,granularity,schedule,seed,"
              "delay_ms,reps,chunk_compute_ms,mean_ms,latency_reduction_pct")


def test_header_is_the_reference_schema():
    assert bc.BENCH_CSV_HEADER == REF_HEADER


def test_row_format_matches_printf_g10():
    cfg = bc.BenchConfig()
    m = bc.BenchMeasurement("fused", 1.0 / 3.0, 12.5)
    assert bc.format_row(cfg, 0.25, m) == "fused,mlp,4,2,64,32,4,1,ring,0,0,10,0.25,0.3333333333,12.5"


def test_latency_reduction_against_first_strategy():
    ms = [bc.BenchMeasurement("baseline", 4.0), bc.BenchMeasurement("data-slicing", 3.0),
          bc.BenchMeasurement("fused", 5.0)]
    bc.latency_reductions(ms)
    assert [m.latency_reduction_pct for m in ms] == [0.0, 25.0, -25.0]


@pytest.mark.parametrize("kw,msg", [
    ({"seq": 63}, "divisible"), ({"granularity": 0}, "granularity"), ({"reps": 0}, "reps"),
    ({"layer": "conv"}, "layer"), ({"schedule": "tree"}, "schedule"),
    ({"schedule": "pairwise", "tp_size": 3, "seq": 63}, "even"),
    ({"layer": "attention", "d_model": 32}, "head_dim"), ({"delay_ms": 1.0}, "delay_ms"),
    ({"seq": 64, "granularity": 32}, "tp_size\\*granularity"),
    ({"layer": "attention", "d_model": 512, "granularity": 2}, "granularity = 1"),
    ({"layer": "ulysses", "heads": 6, "d_model": 768}, "heads \\(6\\) must be divisible"),
    ({"layer": "rs", "granularity": 2, "schedule": "pairwise"}, "ring schedule only")])
def test_validate_rejects(kw, msg):
    with pytest.raises(ValueError, match=msg):
        bc.BenchConfig(**kw).validate()


def test_cli_flags_are_the_config_keys():
    cfg = bc.parse_args(["--layer", "rs", "--tp_size", "2", "--seq", "128", "--schedule", "pairwise"])
    assert (cfg.layer, cfg.tp_size, cfg.seq, cfg.schedule) == ("rs", 2, 128, "pairwise")


@pytest.mark.skipif(not have_reference(), reason="reference oracle not built")
@pytest.mark.parametrize("layer", ["mlp", "rs", "ag", "attention", "ulysses"])
def test_rows_match_reference_run_bench(layer):
    """Same config through the reference's run_bench: identical header, identical strategy
    order, identical config columns; only the three measured columns differ."""
    ref = Reference().bench_csv(layer=layer, reps=1).splitlines()
    cfg = bc.BenchConfig(layer=layer, reps=1)
    res = bc.BenchResult(1.5, [bc.BenchMeasurement(s, 2.0) for s in bc.STRATEGIES])
    bc.latency_reductions(res.measurements)
    mine = bc.format_csv(cfg, res).splitlines()
    assert len(ref) == len(mine) == 4
    assert ref[0] == mine[0]
    for a, b in zip(ref[1:], mine[1:]):
        fa, fb = a.split(","), b.split(",")
        assert len(fa) == len(fb) == 15
        assert fa[:12] == fb[:12], (fa, fb)
        for x in fa[12:]:
            float(x)


@pytest.mark.gpu
@pytest.mark.parametrize("kw", [
    {"layer": "mlp"},                                   # the reference's desk config
    {"layer": "rs", "granularity": 2},
    {"layer": "rs", "schedule": "pairwise"},
    {"layer": "ag", "granularity": 2},
    {"layer": "mlp", "tp_size": 4, "batch": 1, "seq": 2048, "d_model": 1024, "schedule": "circular-slices"},
    {"layer": "attention", "tp_size": 2, "batch": 1, "seq": 512, "d_model": 512, "heads": 4},
    {"layer": "ulysses", "tp_size": 4, "batch": 1, "seq": 1024, "d_model": 512, "heads": 4},
])
def test_gpu_bench_three_strategies(kw):
    """Bench.ThreeStrategiesWithCsvSchema (experiment_test.cpp:172-199) on the B200: three
    measurements in order, the strategies agree on the output (checked inside), CSV schema."""
    import io
    cfg = bc.BenchConfig(reps=2, **kw)
    res = bc.run_bench_collect(cfg)
    assert [m.strategy for m in res.measurements] == list(bc.STRATEGIES)
    assert all(m.mean_ms > 0 for m in res.measurements) and res.chunk_compute_ms > 0
    out = io.StringIO()
    out.write(bc.format_csv(cfg, res))
    lines = out.getvalue().splitlines()
    assert len(lines) == 4 and lines[0] == REF_HEADER
    assert lines[1].startswith(f"baseline,{cfg.layer},{cfg.tp_size},{cfg.batch},{cfg.seq},{cfg.d_model},")
    assert lines[3].startswith(f"fused,{cfg.layer},{cfg.tp_size},")
