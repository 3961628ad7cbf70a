# A/B of the projection's hi*hi segment length at cfg3 (512: 2 segments, 2 TMEM A slots; 1024: one
# segment, 4 A slots), alternated; then the projection-dependent parity tests with the long segment
mkdir -p gpurun_out
for rep in 1 2; do
  timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/seg.log 2>&1
  FKK_PROJECT_SEGLEN=1024 timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/seg.log 2>&1
done
FKK_PROJECT_SEGLEN=256 timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/seg.log 2>&1
grep cfg gpurun_out/seg.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['cfg'], d['env'], {k: round(v,3) for k,v in d['stage_ms_median'].items()}, round(d['total_ms'],3))"
FKK_PROJECT_SEGLEN=1024 timeout 1200 python -m pytest tests -m gpu -q -x -k "projection or cfg3 or factorized or ml_apply or range or conventional or simulation or q_ties" > gpurun_out/seg_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/seg_tests.log
