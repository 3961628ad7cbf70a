mkdir -p gpurun_out
CMD="python tools/run_once.py --workload cfg3 --direct-rows 0"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:project_tc_kernel|reconstruct_tc_kernel|gram_tc_kernel" -c 3 -o gpurun_out/prof_3 $CMD > gpurun_out/ncu_3.log 2>&1; echo ncu=$?
