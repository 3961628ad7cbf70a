# ncu --set full of the three big fKK-EC kernels on cfg3 (one launch each); plain run first.
mkdir -p gpurun_out
CMD="python tools/run_once.py --workload cfg3 --direct-rows 0"
timeout 600 $CMD > gpurun_out/plain_fkk.log 2>&1; echo plain=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:gram_tc_kernel|project_tc_kernel|reconstruct_tc_kernel|tridiag_kernel" -c 4 -o gpurun_out/prof_fkk_cfg3 $CMD > gpurun_out/ncu_full_fkk.log 2>&1; echo ncu=$?; tail -3 gpurun_out/ncu_full_fkk.log
