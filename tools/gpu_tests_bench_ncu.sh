# GPU parity tests + short bench + ncu launch list of one fKK-EC step (used via gpurun)
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 2 --skip-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | cut -c1-1500
CMD="python bench.py --steps 1 --warmup 1 --skip-ml --skip-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu=$?
