# final check of the last session: GPU tests, smoke, default bench line, launch list, ncu --set full of
# the reconstruction (changed epilogue), cfg4 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | cut -c1-300
CMD="python bench.py --steps 1 --warmup 1 --skip-e2e --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; echo ncu_launches=$?
P="python tools/prof_transform.py 262144 1"
timeout 300 $P > gpurun_out/tr_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"reconstruct_tc" -c 1 -o gpurun_out/r2_recon_final -f $P > gpurun_out/ncu_recon.log 2>&1; echo ncu_recon=$?
timeout 2100 python tools/bench_cfg4.py gpurun_out/cfg4.json > gpurun_out/cfg4.log 2>&1; echo cfg4=$?; tail -1 gpurun_out/cfg4.log | cut -c1-300
