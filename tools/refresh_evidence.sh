set -x
P=${P:-r02}
# Evidence refresh on a B200 (run through gpurun): per-GPU table and traces on a cool GPU, the
# bench line, the reference arm, the ncu launch list, ncu --set full of the bench kernels, of the
# per-GPU TP8 virtual ops and of the auxiliary kernels, the no-tail table and the CSV bench.
# Outputs gpurun_out/${P}_*; tools/install_evidence.py copies the summaries into profiles/.
# The auxiliary-kernel ncu capture is ~40 MB: with the other reports it exceeds gpurun's 64 MiB
# copy-back, so it runs in a call of its own: AUX=only runs just that capture, AUX=1 runs both.
aux() {
python tools/ncu_aux.py > gpurun_out/${P}_aux_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"wait_flags|copy_by_parity|softmax_rows|swiglu|ulysses_push|group_kernel" -o gpurun_out/${P}_aux python tools/ncu_aux.py > gpurun_out/${P}_ncu_aux.log 2>&1
}
if [ "${AUX:-0}" = "only" ]; then aux; echo done; exit 0; fi
python tools/perf_virtual.py gpurun_out/${P}_virtual_tp.json > gpurun_out/${P}_pv.log 2>&1
python tools/trace_virtual.py 8 cfg2 steady pairwise > gpurun_out/${P}_trace.log 2>&1
python tools/trace_virtual.py 8 cfg3 steady >> gpurun_out/${P}_trace.log 2>&1
python bench.py > gpurun_out/${P}_bench.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${P}_ref.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${P}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${P}_ncu_launch.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --emulate-tp 0 > gpurun_out/${P}_plain0.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tpf_fused --launch-skip 6 --launch-count 2 -o gpurun_out/${P}_bench_k python bench.py --steps 2 --warmup 3 --no-cpu --emulate-tp 0 > gpurun_out/${P}_ncu_full.log 2>&1
python tools/ncu_virtual_ops.py 8 > gpurun_out/${P}_vops_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tpf_fused -s 6 -c 2 -o gpurun_out/${P}_vops python tools/ncu_virtual_ops.py 8 > gpurun_out/${P}_ncu_vops.log 2>&1
if [ "${AUX:-0}" = "1" ]; then aux; fi
python tools/tail_table.py > gpurun_out/${P}_tail_table.json 2> gpurun_out/${P}_tail.err
bash tools/run_benchcsv.sh gpurun_out/${P}_csv > gpurun_out/${P}_csv.log 2>&1
echo done
