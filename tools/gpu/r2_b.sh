# round-2: GPU tests (all), direct-path timing + stats
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -s > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; grep -E "passed|failed|Error|cfg3 full|cfg4|pair Gram" gpurun_out/gpu_tests.log | tail -15
timeout 300 python tools/prof_direct.py 131072 3 > gpurun_out/direct_time.log 2>&1; echo direct=$?; cat gpurun_out/direct_time.log
