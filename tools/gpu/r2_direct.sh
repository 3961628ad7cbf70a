# direct-path parity tests + timing (+ ncu --set full of the direct kernels after a plain run of the same command)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -m gpu -q -x -k "direct or floor or iteration or wide or cfg4" > gpurun_out/gpu_direct_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_direct_tests.log
timeout 300 python tools/prof_direct.py 131072 3 > gpurun_out/direct_time.log 2>&1; echo direct=$?; cat gpurun_out/direct_time.log
if [ "$1" = "ncu" ]; then
P="python tools/prof_direct.py 32768 1"
timeout 300 $P > gpurun_out/direct_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"direct_phase|als_seg|direct_finish" -c 3 -o gpurun_out/r2_direct3 -f $P > gpurun_out/ncu_direct.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_direct.log
fi
