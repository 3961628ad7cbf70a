mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host" > gpurun_out/host_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/host_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_e2e.log 2>&1; echo bench=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_e2e.log').read().strip().splitlines()[-1])
print(json.dumps(d['e2e']))
PY
