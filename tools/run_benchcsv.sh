#!/bin/bash
# Dev / evidence tool: the three-strategy bench in the reference's CSV schema on one B200
# (single-GPU local group), at BASELINE-sized shapes. Usage: tools/run_benchcsv.sh OUTDIR
set -e
out=${1:-gpurun_out}
mkdir -p "$out"
py() { python -m paper_2604_24013_b200.benchcsv "$@"; }
{
  py --layer mlp --tp_size 4 --batch 1 --seq 8192 --d_model 4096 --reps 10
  py --layer mlp --tp_size 8 --batch 1 --seq 8192 --d_model 4096 --reps 10 --schedule pairwise | tail -n +2
  py --layer rs --tp_size 4 --batch 1 --seq 8192 --d_model 4096 --reps 10 | tail -n +2
  py --layer ag --tp_size 4 --batch 1 --seq 8192 --d_model 4096 --reps 10 | tail -n +2
  py --layer attention --tp_size 4 --batch 1 --seq 8192 --d_model 4096 --heads 32 --reps 5 | tail -n +2
  py --layer ulysses --tp_size 8 --batch 1 --seq 32768 --d_model 4096 --heads 32 --reps 3 | tail -n +2
} > "$out/bench_csv.csv"
cat "$out/bench_csv.csv"
