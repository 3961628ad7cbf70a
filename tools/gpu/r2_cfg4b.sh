# BASELINE configs[3] (cfg4: 4,000,000 x 1600, k = 100) on one B200 after the Gram-split / ridge fixes
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/cfg4_smi.txt 2>&1
timeout 2100 python tools/bench_cfg4.py gpurun_out/cfg4.json > gpurun_out/cfg4.log 2>&1; echo cfg4=$?; tail -1 gpurun_out/cfg4.log | cut -c1-700
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> gpurun_out/cfg4_smi.txt 2>&1
