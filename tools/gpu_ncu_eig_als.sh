mkdir -p gpurun_out
python tools/run_once.py --workload cfg2 --rows 4096 --direct-rows 8192 > gpurun_out/plain_als.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k "regex:als_part_kernel" -c 1 -o gpurun_out/prof_als python tools/run_once.py --workload cfg2 --rows 4096 --direct-rows 8192 > gpurun_out/ncu_als.log 2>&1; echo ncu_als=$?
python tools/eig_breakdown.py 1000 60 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k "regex:tridiag_rows_kernel|backxform_reg" -c 2 -o gpurun_out/prof_eig python tools/eig_breakdown.py 1000 60 > gpurun_out/ncu_eig.log 2>&1; echo ncu_eig=$?
timeout 300 python -m pytest tests/test_gpu_eig.py -q -x 2>&1 | tail -2
