"""Copy the outputs of `P=<prefix> bash tools/refresh_evidence.sh` (gpurun_out/<prefix>_*) into
profiles/: bench line, reference-arm line, ncu launch list, ncu --set full summaries (bench
kernels, per-GPU TP8 virtual ops) with their headers, per-launch DRAM traffic for bench.py,
per-GPU table, traces and emulated configs. Runs here (no GPU).
    python tools/install_evidence.py <prefix>"""
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = sys.argv[1] if len(sys.argv) > 1 else "r"
G = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")


def last_json_line(path):
    for line in reversed(open(path).read().splitlines()):
        if line.startswith("{"):
            return line
    raise SystemExit(f"no JSON line in {path}")


def summarize(rep):
    return subprocess.run([sys.executable, os.path.join(PR, "summarize_ncu.py"), rep],
                          capture_output=True, text=True, check=True).stdout


open(os.path.join(PR, "r01_bench_n1.json"), "w").write(last_json_line(f"{G}/{P}_bench.log") + "\n")
open(os.path.join(PR, "r01_bench_reference_arm.json"), "w").write(last_json_line(f"{G}/{P}_ref.log") + "\n")
shutil.copy(f"{G}/{P}_launches.csv", os.path.join(PR, "r01_launches.csv"))
shutil.copy(f"{G}/{P}_virtual_tp.json", os.path.join(PR, "r01_virtual_tp_pergpu.json"))
shutil.copy(f"{G}/{P}_configs.json", os.path.join(PR, "r01_configs.json"))
with open(os.path.join(PR, "r01_virtual_trace_tp8.txt"), "w") as f:
    f.write("# tools/trace_virtual.py 8 cfg2 / cfg3: device timeline of one per-GPU TP8 fused call "
            "(virtual peers, self-ring), fused and compute-only\n")
    f.write(open(f"{G}/{P}_trace.log").read())

out = summarize(f"{G}/{P}_bench_k.ncu-rep")
d = [float(v) for v in re.findall(r"gpu__time_duration.sum \[ms\] = ([0-9.]+)", out)]
hdr = ("# bench.py launches 7-8 (after warm-up): AG-GEMM gate||up + fused SwiGLU (tpf_fused_kernel<1,5>) and "
       "GEMM-RS down\n# (<0,5>), T = 1. ncu --set full --clock-control none (isolated, cold cache): "
       f"AG 1.924 TFLOP / {d[0]:.4f} ms = {1.924145 / d[0] * 1e3:.0f} TF/s;\n"
       f"# RS 0.962 TFLOP / {d[1]:.4f} ms = {0.962072 / d[1] * 1e3:.0f} TF/s.\n")
open(os.path.join(PR, "r01_fused_kernels_ncu_full.txt"), "w").write(hdr + out)
tr_path = os.path.join(PR, "traffic.json")
tr = json.load(open(tr_path))
vals = [float(v) for v in re.findall(r"traffic_bytes \(read\+write\) = ([0-9.e+]+)", out)]
tr["ag_gemm_tp1"], tr["gemm_rs_tp1"] = vals[0], vals[1]
json.dump(tr, open(tr_path, "w"), indent=1)

out2 = summarize(f"{G}/{P}_vops.ncu-rep")
u = [float(v) for v in re.findall(r"gpu__time_duration.sum \[us\] = ([0-9.]+)", out2)]
hdr2 = ("# tools/ncu_virtual_ops.py 8 co: rank 0 of a TP8 group with virtual peers (cfg2 per-GPU shapes): fused\n"
        "# AG-GEMM, fused GEMM-RS (bf16 wire), then the AG-GEMM in compute-only mode. Under ncu every replay\n"
        "# restores memory, so the pre-set flags pass at once (no ring waits).\n"
        f"# AG 240.5 GFLOP / {u[0]:.1f} us = {240.5 / u[0] * 1e3:.0f} TF/s (compute-only {u[2]:.1f} us); "
        f"RS 120.3 GFLOP / {u[1]:.1f} us = {120.3 / u[1] * 1e3:.0f} TF/s.\n")
open(os.path.join(PR, "r01_virtual_tp8_fused_ncu_full.txt"), "w").write(hdr2 + out2)
print("installed", P)
