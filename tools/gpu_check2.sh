mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/gpu_tests.log
python tools/eig_breakdown.py 1000 60 2>&1 | grep ms
timeout 300 python tools/time_eig.py cfg3 > gpurun_out/time_eig.log 2>&1; echo time=$?; tail -3 gpurun_out/time_eig.log
timeout 300 python bench.py --steps 2 --warmup 1 --skip-ml --skip-e2e --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_quick.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stage_ms'], d['direct_kk'])"
