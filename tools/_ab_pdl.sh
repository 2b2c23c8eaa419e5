python tools/ab_env.py "TPF_PDL_FUSED=0" "TPF_PDL_FUSED=1" --rounds 4 > gpurun_out/ab_pdl.txt 2>&1
TPF_PDL_FUSED=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_split.py -q -x -k "c1 or fuzz or repeated" > gpurun_out/t_pdl.log 2>&1; echo rc=$? >> gpurun_out/t_pdl.log
