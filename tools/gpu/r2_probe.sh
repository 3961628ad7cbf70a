# round-2 probe: GPU tests, direct-path timing, ncu --set full of the direct kernels (+source)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
timeout 300 python tools/prof_direct.py 131072 3 > gpurun_out/direct_time.log 2>&1; echo direct=$?; cat gpurun_out/direct_time.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"direct_phase|als_part|direct_finish" -c 3 -o gpurun_out/r2_direct python tools/prof_direct.py 32768 1 > gpurun_out/ncu_direct.log 2>&1; echo ncu=$?; tail -3 gpurun_out/ncu_direct.log
