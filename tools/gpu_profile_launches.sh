timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "cfg2" > gpurun_out/gpu_tests_cfg2.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests_cfg2.log
CMD="python bench.py --steps 1 --warmup 1 --skip-ml --skip-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu3.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu3.log
