mkdir -p gpurun_out
CMD="python tools/run_once.py --workload cfg3 --direct-rows 0"
# (the pair kernel is the default at M = 1000)
timeout 600 $CMD > gpurun_out/plain_g2.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:gram_pre2" -c 1 -o gpurun_out/prof_g2 $CMD > gpurun_out/ncu_g2.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_g2.ncu-rep --page source --csv --print-source sass > gpurun_out/g2_src.csv 2>/dev/null
