# dev sweep: raster for the T = 1 GEMMs without hints (timing, then ncu DRAM bytes)
run() { env "$@" python tools/l2_probe.py $OP >> gpurun_out/l2_time.txt 2>&1; }
prof() { env "$@" PROBE_N=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tpf_fused -s 3 -c 1 --csv python tools/l2_probe.py $OP 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' -v tag="$OP $*" '{print tag, $(NF-2), $NF}' >> gpurun_out/l2_ncu.txt; }
rm -f gpurun_out/l2_time.txt gpurun_out/l2_ncu.txt
OP=rs; for cfg in "X=0" "TPF_GROUP_N=16" "TPF_GROUP_N=8" "TPF_GROUP_N=4" "TPF_GROUP_N=2" "TPF_GROUP_N=8 TPF_L2_B=2" "TPF_GROUP_N=8 TPF_L2_A=1"; do run $cfg; run $cfg; prof $cfg; done
OP=ag; for cfg in "X=0" "TPF_GROUP_M=12" "TPF_GROUP_M=24" "TPF_L2_A=2" "TPF_L2_B=1"; do run $cfg; run $cfg; prof $cfg; done
