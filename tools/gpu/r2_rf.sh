mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_r2.py -m gpu -q -x -s -k "range_finder or wide" > gpurun_out/gpu_rf_tests.log 2>&1; echo tests=$?; grep -E "passed|failed|Error|range finder|assert" gpurun_out/gpu_rf_tests.log | tail -12
timeout 900 python bench.py --steps 5 --warmup 2 --skip-e2e --no-cpu-baseline > gpurun_out/bench_rf.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_rf.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({k:d[k] for k in ('value','ms_per_step','stage_ms','range_finder','ml_apply')})[:3000])"
