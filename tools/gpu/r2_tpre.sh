# A/B of the WY back-transformation: T rows loaded before the block's dots and barrier (default)
# against after it (FKK_BX_TPRE=0), alternated; then the eig / transform parity tests
mkdir -p gpurun_out
for rep in 1 2; do
  FKK_BX_TPRE=0 timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/tpre.log 2>&1
  timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/tpre.log 2>&1
done
grep cfg gpurun_out/tpre.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['env'], {k: round(v,3) for k,v in d['stage_ms_median'].items()}, round(d['total_ms'],3))"
timeout 1200 python -m pytest tests -m gpu -q -x -k "eig or cfg3 or factorized or range or conventional or ml_apply or simulation" > gpurun_out/tpre_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/tpre_tests.log
