set -x
P=${P:-r}
# Evidence refresh on a B200 (run through gpurun): bench line, reference arm, ncu launch list,
# ncu --set full of the bench kernels and of the per-GPU TP8 virtual ops, per-GPU table, traces,
# emulated configs. Outputs gpurun_out/${P}_*; copy the summaries into profiles/.
# per-GPU table first, on a cool GPU: after the bench's sustained load the same calls run up to 30% slower
python tools/perf_virtual.py gpurun_out/${P:-r}_virtual_tp.json > gpurun_out/${P:-r}_pv.log 2>&1
python bench.py > gpurun_out/${P:-r}_bench.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${P:-r}_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P:-r}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${P:-r}_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tpf_fused --launch-skip 6 --launch-count 2 -o gpurun_out/${P:-r}_bench_k python bench.py --steps 2 --warmup 3 --no-cpu --emulate-tp 0 > gpurun_out/${P:-r}_ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tpf_fused -o gpurun_out/${P:-r}_vops python tools/ncu_virtual_ops.py 8 co > gpurun_out/${P:-r}_ncu_vops.log 2>&1
python tools/trace_virtual.py 8 cfg2 > gpurun_out/${P:-r}_trace.log 2>&1
python tools/trace_virtual.py 8 cfg3 >> gpurun_out/${P:-r}_trace.log 2>&1
timeout 900 python tools/perf_configs.py gpurun_out/${P:-r}_configs.json > gpurun_out/${P:-r}_cfg.log 2>&1
echo done
