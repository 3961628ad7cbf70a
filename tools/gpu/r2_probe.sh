# multicast probe + ALS timing/parity of the current build
mkdir -p gpurun_out
./tools/micro/mcprobe > gpurun_out/mcprobe.log 2>&1; echo mcprobe=$?; cat gpurun_out/mcprobe.log
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1; head -5 gpurun_out/topo.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "direct or conventional or als or wide or paper" > gpurun_out/als_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/als_tests.log
timeout 600 python tools/prof_direct.py 703026 3 2>&1 | grep -v Warn
