mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:inviter_kernel|backxform" -c 2 -o gpurun_out/prof_bis python tools/eig_breakdown.py 1000 60 > gpurun_out/ncu_bis.log 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_bis.ncu-rep --page source --csv --print-source sass > gpurun_out/bis_src.csv 2>/dev/null
