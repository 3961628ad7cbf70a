# full run: all GPU tests, smoke, bench, launch list, ncu --set full of the direct kernels (final code)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | cut -c1-300
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu_launches=$?
P="python tools/prof_direct.py 32768 1"
timeout 300 $P > gpurun_out/direct_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"direct_phase|als_seg|direct_finish" -c 3 -o gpurun_out/r2_direct_final -f $P > gpurun_out/ncu_direct.log 2>&1; echo ncu_direct=$?
