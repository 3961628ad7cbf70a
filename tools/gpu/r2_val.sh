# validation of HEAD: GPU tests, smoke, bench line, ncu source capture of the two FFT kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | cut -c1-400
P="python tools/prof_direct.py 32768 1"
timeout 300 $P > gpurun_out/direct_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"direct_phase|direct_finish" -c 2 -o gpurun_out/r2_fft_src -f $P > gpurun_out/ncu_fft.log 2>&1; echo ncu_fft=$?
