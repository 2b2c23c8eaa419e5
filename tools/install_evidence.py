"""Copy the outputs of `P=<prefix> bash tools/refresh_evidence.sh` (gpurun_out/<prefix>_*) into
profiles/<prefix>_*: bench line, reference-arm line, ncu launch list, ncu --set full summaries
(bench kernels, per-GPU TP8 virtual ops, auxiliary kernels) with their headers, per-launch DRAM
traffic for bench.py, per-GPU table, traces, tail table and CSV bench. Runs here (no GPU).
    python tools/install_evidence.py <prefix>"""
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = sys.argv[1] if len(sys.argv) > 1 else "r02"
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


def have(path):
    ok = os.path.exists(path)
    if not ok:
        print("missing", path)
    return ok


if have(f"{G}/{P}_bench.log"):
    open(os.path.join(PR, f"{P}_bench_n1.json"), "w").write(last_json_line(f"{G}/{P}_bench.log") + "\n")
if have(f"{G}/{P}_ref.log"):
    open(os.path.join(PR, f"{P}_bench_reference_arm.json"), "w").write(last_json_line(f"{G}/{P}_ref.log") + "\n")
for src, dst in ((f"{P}_launches.csv", f"{P}_launches.csv"), (f"{P}_virtual_tp.json", f"{P}_virtual_tp_pergpu.json"),
                 (f"{P}_tail_table.json", f"{P}_tail_table.json"), (f"{P}_csv/bench_csv.csv", f"{P}_bench_csv.csv")):
    if have(f"{G}/{src}"):
        shutil.copy(f"{G}/{src}", os.path.join(PR, dst))
if have(f"{G}/{P}_trace.log"):
    with open(os.path.join(PR, f"{P}_virtual_trace_tp8.txt"), "w") as f:
        f.write("# tools/trace_virtual.py 8 cfg2|cfg3 steady [pairwise]: device timeline of one per-GPU TP8 fused call\n"
                "# (virtual peers, self-ring) traced between back-to-back calls; fused and compute-only\n")
        f.write(open(f"{G}/{P}_trace.log").read())

if have(f"{G}/{P}_bench_k.ncu-rep"):
    out = summarize(f"{G}/{P}_bench_k.ncu-rep")
    d = [float(v) for v in re.findall(r"gpu__time_duration.sum \[ms\] = ([0-9.]+)", out)]
    hdr = ("# bench.py --emulate-tp 0, launches 7-8 (after warm-up): AG-GEMM gate||up + fused SwiGLU "
           "(tpf_fused_kernel<1,5>) and GEMM-RS down\n# (<0,5>), T = 1. ncu --set full --clock-control none "
           f"(isolated, cold cache): AG 1.924 TFLOP / {d[0]:.4f} ms = {1.924145 / d[0] * 1e3:.0f} TF/s;\n"
           f"# RS 0.962 TFLOP / {d[1]:.4f} ms = {0.962072 / d[1] * 1e3:.0f} TF/s. Tensor-pipe note: for these\n"
           "# cta_group::2 kernels sm__pipe_tensor_cycles_active does not track the FLOP rate (DESIGN 4c);\n"
           "# use sm__mem_tensor_cycles_active or the FLOP rate.\n")
    open(os.path.join(PR, f"{P}_fused_kernels_ncu_full.txt"), "w").write(hdr + out)
    tr_path = os.path.join(PR, "traffic.json")
    tr = json.load(open(tr_path))
    vals = [float(v) for v in re.findall(r"traffic_bytes \(read\+write\) = ([0-9.e+]+)", out)]
    tr["ag_gemm_tp1"], tr["gemm_rs_tp1"] = vals[0], vals[1]
    tr["source"] = (f"ncu --set full (profiles/{P}_fused_kernels_ncu_full.txt): dram__bytes_read.sum + "
                    "dram__bytes_write.sum per launch, bench.py --steps 2 --warmup 3 --emulate-tp 0 "
                    "(launches 7-8: AG-GEMM gate||up+SwiGLU, GEMM-RS down), current build")
    json.dump(tr, open(tr_path, "w"), indent=1)

if have(f"{G}/{P}_vops.ncu-rep"):
    out2 = summarize(f"{G}/{P}_vops.ncu-rep")
    u = [float(v) for v in re.findall(r"gpu__time_duration.sum \[us\] = ([0-9.]+)", out2)]
    hdr2 = ("# tools/ncu_virtual_ops.py 8, ncu -s 6 -c 2: the fourth fused AG-GEMM and GEMM-RS (bf16 wire) of rank 0\n"
            "# of a TP8 group with virtual peers (cfg2 per-GPU shapes). Replays restore memory to the state before\n"
            "# the profiled launch, where the flags hold the previous call's epoch: the ring waits are real.\n"
            f"# AG 240.5 GFLOP / {u[0]:.1f} us = {240.5 / u[0] * 1e3:.0f} TF/s; "
            f"RS 120.3 GFLOP / {u[1]:.1f} us = {120.3 / u[1] * 1e3:.0f} TF/s.\n")
    open(os.path.join(PR, f"{P}_virtual_tp8_fused_ncu_full.txt"), "w").write(hdr2 + out2)

if have(f"{G}/{P}_aux.ncu-rep"):
    out3 = summarize(f"{G}/{P}_aux.ncu-rep")
    hdr3 = ("# tools/ncu_aux.py: one launch of each auxiliary kernel, ncu --set full --clock-control none: the flag\n"
            "# waits (wait_flags, wait_flags2), the parity-selected copy (copy_by_parity), the unfused attention's\n"
            "# softmax (softmax_rows), the Ulysses push, the unfused SwiGLU, and the split-group GEMM kernel\n"
            "# (tpf_fused_group_kernel: four ranks' per-process launches in one grid).\n")
    open(os.path.join(PR, f"{P}_aux_kernels_ncu_full.txt"), "w").write(hdr3 + out3)
print("installed", P)
