mkdir -p gpurun_out
CMD="python tools/kernel_breakdown.py --what direct --rows 65536 --reps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:als_part|direct_phase|direct_finish" -c 3 -o gpurun_out/prof_direct2 $CMD > gpurun_out/ncu_direct2.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_direct2.log
