mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -4 gpurun_out/gpu_tests.log
timeout 300 python tools/time_eig.py cfg3 > gpurun_out/time_eig.log 2>&1; echo time=$?; tail -3 gpurun_out/time_eig.log
CMD="python tools/run_once.py --workload cfg3 --direct-rows 0"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:project_tc_kernel|reconstruct_tc_kernel" -c 2 -o gpurun_out/prof_pr $CMD > gpurun_out/ncu_pr.log 2>&1; echo ncu=$?
