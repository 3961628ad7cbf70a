mkdir -p gpurun_out
CMD="python tools/run_once.py --workload cfg2 --direct-rows 65536"
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:direct_phase|direct_finish" -c 2 -o gpurun_out/prof_dp $CMD > gpurun_out/ncu_dp.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_dp.ncu-rep --page source --csv --print-source sass -k regex:direct_phase > gpurun_out/dp_src.csv 2>/dev/null
ncu -i gpurun_out/prof_dp.ncu-rep --page source --csv --print-source sass -k regex:direct_finish > gpurun_out/df_src.csv 2>/dev/null
