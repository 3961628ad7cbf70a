mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_r2.py -m gpu -q -x -s -k "paper_simulation" > gpurun_out/gpu_sim_test.log 2>&1; echo tests=$?; grep -E "passed|failed|paper sim|Error|assert" gpurun_out/gpu_sim_test.log | tail -5
timeout 1500 python tools/paper_sim.py gpurun_out/paper_sim.json > gpurun_out/paper_sim.log 2>&1; echo sim=$?; tail -6 gpurun_out/paper_sim.log | cut -c1-700
