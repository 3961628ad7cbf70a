# eigensolver kernels at M = 1600 (cfg4 geometry): launch times and the tridiagonalisation's counters
mkdir -p gpurun_out
P="python tools/prof_cfg4.py 65536 1"
timeout 300 $P > gpurun_out/e16_plain.log 2>&1; tail -1 gpurun_out/e16_plain.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e16_launches.csv $P > gpurun_out/e16_ncu.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none -k regex:"tridiag_rows" -c 1 -o gpurun_out/e16_tridiag -f $P > gpurun_out/e16_ncu2.log 2>&1; echo full=$?
