# full ncu captures of the hot kernels of one cfg3 transform (for profiles/)
mkdir -p gpurun_out
CMD="python tools/run_once.py --workload cfg3 --direct-rows 0"
timeout 600 $CMD > gpurun_out/plain_round.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:gram_pre2_kernel|logratio_pre_kernel|project_tma_kernel|reconstruct_tc_kernel|tridiag_rows_kernel" -c 5 -o gpurun_out/prof_round $CMD > gpurun_out/ncu_round.log 2>&1; echo ncu=$?
