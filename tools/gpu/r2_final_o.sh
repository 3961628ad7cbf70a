# final check of the round at HEAD (after the WY back-transformation change): GPU tests, smoke, default bench
# line, launch list, ncu --set full of backxform_wy (the changed kernel) at cfg3 geometry
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | cut -c1-300
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu_launches=$?
P="python tools/prof_transform.py 262144 1"
timeout 300 $P > gpurun_out/tr_plain.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:"backxform_wy" -c 1 -o gpurun_out/r2_backxform_final -f $P > gpurun_out/ncu_backxform.log 2>&1; echo ncu_backxform=$?
