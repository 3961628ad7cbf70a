# A/B of the reconstruction chunk width (FKK_RT_NCH) at cfg4 geometry (k = 100) and cfg3, then the
# parity tests that reach the reconstruction
mkdir -p gpurun_out
for v in 16 32; do
  FKK_RT_NCH=$v timeout 300 python tools/time_stages.py cfg4 1000000 5 >> gpurun_out/nch.log 2>&1
done
timeout 300 python tools/time_stages.py cfg4 1000000 5 >> gpurun_out/nch.log 2>&1
timeout 300 python tools/time_stages.py cfg3 703026 9 >> gpurun_out/nch.log 2>&1
grep cfg gpurun_out/nch.log | cut -c1-400
timeout 900 python -m pytest tests -m gpu -q -x -k "cfg4 or factorized or ml_apply or conventional or cfg3 or host" > gpurun_out/nch_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/nch_tests.log
