mkdir -p gpurun_out
CMD="python tools/run_once.py --workload cfg3 --direct-rows 0"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:logratio_pre|gram_pre" -c 2 -o gpurun_out/prof_lp $CMD > gpurun_out/ncu_lp.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_lp.log
