# A/B of the eig stage: WY-factor kernel on a forked stream (default) against in order
# (FKK_WYT_FORK=0), alternated; bisection CTA width; then the eig / transform parity tests
mkdir -p gpurun_out
for rep in 1 2; do
  FKK_WYT_FORK=0 timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/wyt.log 2>&1
  timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/wyt.log 2>&1
done
FKK_BISECT_THREADS=256 timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/wyt.log 2>&1
FKK_BISECT_THREADS=64 timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/wyt.log 2>&1
grep cfg gpurun_out/wyt.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['env'], {k: round(v,3) for k,v in d['stage_ms_median'].items()}, round(d['total_ms'],3))"
timeout 1200 python -m pytest tests -m gpu -q -x -k "eig or cfg3 or cfg4 or factorized or range or nccl" > gpurun_out/wyt_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/wyt_tests.log
