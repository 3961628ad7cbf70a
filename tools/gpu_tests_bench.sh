# GPU parity tests + smoke + short bench (used via gpurun)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 2 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?; tail -3 gpurun_out/bench.log
