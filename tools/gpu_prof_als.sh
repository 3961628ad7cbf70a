mkdir -p gpurun_out
CMD="python tools/run_once.py --workload cfg2 --direct-rows 65536"
timeout 600 $CMD > gpurun_out/plain_als.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:als_part_kernel|direct_phase|direct_finish" -c 3 -o gpurun_out/prof_als $CMD > gpurun_out/ncu_als.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_als.ncu-rep --page source --csv --print-source sass -k regex:als_part > gpurun_out/als_src.csv 2>/dev/null
ncu -i gpurun_out/prof_als.ncu-rep --page source --csv --print-source sass -k regex:direct_finish > gpurun_out/fin_src.csv 2>/dev/null
