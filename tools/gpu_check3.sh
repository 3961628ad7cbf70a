mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -4 gpurun_out/gpu_tests.log
timeout 300 python tools/time_eig.py cfg3 > gpurun_out/time_eig.log 2>&1; echo time=$?; tail -3 gpurun_out/time_eig.log
