# ncu --set full of the projection and reconstruction kernels (cfg3 geometry, 262,144 rows)
mkdir -p gpurun_out
P="python tools/prof_transform.py 262144 1"
timeout 300 $P > gpurun_out/tr_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"reconstruct_tc|project_tma" -c 2 -o gpurun_out/r2_recon -f $P > gpurun_out/ncu_recon.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_recon.log
