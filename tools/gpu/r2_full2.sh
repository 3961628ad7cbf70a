# all GPU tests, smoke, the default bench line, launch list of one bench step, ncu --set full of the hot
# fKK-EC kernels (traffic), each ncu only after the same command exited 0 without it
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -s > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; grep -E "passed|failed|Error|cfg3 full|cfg4|pair Gram|range finder" gpurun_out/gpu_tests.log | tail -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | cut -c1-600
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu_launches=$?
T="python tools/prof_transform.py 703026 1"
timeout 300 $T > gpurun_out/prof_t_plain.log 2>&1 && timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"gram_pre2|project_tma|reconstruct_tc|logratio_pre|tridiag_rows" -c 5 -o gpurun_out/r2_fkk_full -f $T > gpurun_out/ncu_fkk.log 2>&1; echo ncu_full=$?
