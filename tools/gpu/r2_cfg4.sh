# BASELINE configs[3] (cfg4: 4,000,000 x 1600, k = 100) on one B200: fKK-EC transform + direct pass;
# then the cfg4-geometry parity tests
mkdir -p gpurun_out
timeout 2100 python tools/bench_cfg4.py gpurun_out/cfg4.json > gpurun_out/cfg4.log 2>&1; echo cfg4=$?; tail -1 gpurun_out/cfg4.log | cut -c1-700
timeout 900 python -m pytest tests -m gpu -q -x -k "cfg4 or odd_channel or wide or image_gram or gram" > gpurun_out/cfg4_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/cfg4_tests.log
