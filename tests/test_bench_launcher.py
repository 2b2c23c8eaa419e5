"""bench.py's multi-GPU launcher on CPU (gloo): `--gpus N` without a torchrun environment
launches N ranks itself (torch.distributed.run on 127.0.0.1), rank 0 prints exactly one JSON
line with n_gpus == N, and a world size that disagrees with --gpus is refused."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env(**kw):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    env.update(kw)
    return env


def test_bench_gpus_2_launches_two_ranks_and_prints_one_line():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "3"],
                       capture_output=True, text=True, timeout=300, env=_env(), cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ranks_seen"] == 2 and d["dry_run"] is True and d["steps"] == 3


def test_bench_refuses_world_size_mismatch():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=_env(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"),
                       cwd=ROOT)
    assert p.returncode == 2 and "WORLD_SIZE=2" in p.stderr
