# ncu --set full of the streaming kernels of the headline transform (projection, reconstruction, log-ratio pre-pass)
mkdir -p gpurun_out
P="python tools/prof_transform.py 703026 1"
timeout 300 $P > gpurun_out/transform_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"project_tma|reconstruct_tc|logratio_pre" -c 3 -o gpurun_out/r2_stream -f $P > gpurun_out/ncu_stream.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_stream.log
