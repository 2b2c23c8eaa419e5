set -x
python bench.py > gpurun_out/f_bench.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/f_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tpf_fused --launch-skip 6 --launch-count 2 -o gpurun_out/f_bench_k python bench.py --steps 2 --warmup 3 --no-cpu --emulate-tp 0 > gpurun_out/f_ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tpf_fused -o gpurun_out/f_vops python tools/ncu_virtual_ops.py 8 co > gpurun_out/f_ncu_vops.log 2>&1
python tools/perf_virtual.py gpurun_out/f_virtual_tp.json > gpurun_out/f_pv.log 2>&1
python tools/trace_virtual.py 8 cfg2 > gpurun_out/f_trace.log 2>&1
python tools/trace_virtual.py 8 cfg3 >> gpurun_out/f_trace.log 2>&1
timeout 900 python tools/perf_configs.py gpurun_out/f_configs.json > gpurun_out/f_cfg.log 2>&1
echo done
