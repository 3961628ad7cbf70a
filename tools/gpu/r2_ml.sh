mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --skip-e2e --no-cpu-baseline > gpurun_out/bench_ml.log 2>&1; echo bench=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_ml.log').read().strip().splitlines()[-1])
m=d['ml_apply']; print({k: m[k] for k in ('ms_per_batch','ms_per_batch_one_stream','streams')}, m['roofline']['frac'])
print('gram', d['stage_ms']['gram'], 'ms/step', d['ms_per_step'], 'frac', d['roofline']['frac'])
PY
