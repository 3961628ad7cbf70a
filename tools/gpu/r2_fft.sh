# ncu --set full of the direct-path FFT kernels (phase, finish) after a plain run of the same command
mkdir -p gpurun_out
P="python tools/prof_direct.py 32768 1"
timeout 300 $P > gpurun_out/direct_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"direct_phase|direct_finish" -c 2 -o gpurun_out/r2_fft -f $P > gpurun_out/ncu_fft.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_fft.log
