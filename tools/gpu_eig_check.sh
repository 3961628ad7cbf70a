mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_eig.py -q -x > gpurun_out/eig_tests.log 2>&1; echo eigtests=$?; tail -15 gpurun_out/eig_tests.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -5 gpurun_out/gpu_tests.log
timeout 300 python tools/time_eig.py cfg3 > gpurun_out/time_eig.log 2>&1; echo time=$?; tail -3 gpurun_out/time_eig.log
