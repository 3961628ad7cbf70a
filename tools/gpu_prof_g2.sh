mkdir -p gpurun_out
CMD="python tools/run_once.py --workload cfg3 --direct-rows 0"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:gram_pre2_kernel" -c 1 -o gpurun_out/prof_g2 $CMD > gpurun_out/ncu_g2.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_g2.log
