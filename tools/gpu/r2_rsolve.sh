# A/B of the eigensolver's CholQR2 apply: forward substitution with R (default) against the explicit
# inverse (FKK_CHOLQR_SOLVE=0), alternated; then every GPU test
mkdir -p gpurun_out
for rep in 1 2; do
  FKK_CHOLQR_SOLVE=0 timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/rsolve.log 2>&1
  timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/rsolve.log 2>&1
done
grep cfg gpurun_out/rsolve.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['env'], {k: round(v,3) for k,v in d['stage_ms_median'].items()}, round(d['total_ms'],3))"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/rsolve_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/rsolve_tests.log
