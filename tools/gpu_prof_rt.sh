mkdir -p gpurun_out
CMD="python tools/run_once.py --workload cfg3 --direct-rows 0"
timeout 600 $CMD > gpurun_out/plain_rt.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:reconstruct_tc_kernel" -c 1 -o gpurun_out/prof_rt $CMD > gpurun_out/ncu_rt.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_rt.ncu-rep --page source --csv --print-source sass > gpurun_out/rt_src.csv 2>/dev/null
