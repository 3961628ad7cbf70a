# TMEM ALS: direct-path parity tests, timing of the direct pass at cfg3 size, ncu of the ALS kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "direct or conventional or als or wide or paper" > gpurun_out/als_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/als_tests.log
timeout 600 python tools/prof_direct.py 703026 3 2>&1 | grep -v Warn
if [ "$1" = "ncu" ]; then
P="python tools/prof_direct.py 32768 1"
timeout 300 $P > gpurun_out/direct_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"als_seg" -c 1 -o gpurun_out/r2_als_tmem -f $P > gpurun_out/ncu_als.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_als.log
fi
