# A/B of the reconstruction epilogue: one chunk per step (FKK_RT_PAIR=0) against chunk pairs (default
# where the smem fits: cfg3), alternated; cfg4 geometry; then the GPU parity tests
mkdir -p gpurun_out
for rep in 1 2; do
  FKK_RT_PAIR=0 timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/pair.log 2>&1
  timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/pair.log 2>&1
done
timeout 300 python tools/time_stages.py cfg4 1000000 5 >> gpurun_out/pair.log 2>&1
grep cfg gpurun_out/pair.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['env'], {k: round(v,3) for k,v in d['stage_ms_median'].items()}, round(d['total_ms'],3))"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pair_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/pair_tests.log
