# ncu --set full of the fKK-EC kernels on the final code (cfg3, full image, one transform)
mkdir -p gpurun_out
P="python tools/prof_transform.py 703026 1"
timeout 300 $P > gpurun_out/fkk_plain.log 2>&1; tail -1 gpurun_out/fkk_plain.log | cut -c1-200
timeout 1500 ncu --set full --clock-control none -k regex:"logratio_pre|gram_pre2|tridiag_rows|project_tma|reconstruct_tc" -c 5 -o gpurun_out/r2_fkk_final -f $P > gpurun_out/ncu_fkk.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_fkk.log
