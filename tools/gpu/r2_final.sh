# final check: bench line (clock sampling fix) + the reference arm
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_final.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref.log 2>&1; echo ref=$?; tail -1 gpurun_out/ref.log | cut -c1-400
