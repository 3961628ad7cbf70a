mkdir -p gpurun_out
CMD="python tools/run_once.py --workload cfg2 --direct-rows 0"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ridge_factor" -c 1 -o gpurun_out/prof_ridge $CMD > gpurun_out/ncu_ridge.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_ridge.ncu-rep --page source --csv --print-source sass > gpurun_out/ridge_src.csv 2>/dev/null
