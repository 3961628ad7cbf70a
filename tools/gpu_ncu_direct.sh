mkdir -p gpurun_out
CMD="python tools/run_once.py --workload cfg2 --rows 4096 --direct-rows 32768"
$CMD > gpurun_out/plain_direct.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k "regex:als_part_kernel<float|direct_phase|direct_finish" -c 3 -o gpurun_out/prof_direct $CMD > gpurun_out/ncu_direct.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_direct.log
