# ML apply: batches over 2 / 3 / 4 streams (bench's ml_apply leg only)
mkdir -p gpurun_out
for ns in 2 3 4; do FKK_BENCH_ML_STREAMS=$ns timeout 900 python bench.py --steps 3 --warmup 3 --skip-e2e --no-cpu-baseline > gpurun_out/ml_$ns.log 2>&1; tail -1 gpurun_out/ml_$ns.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); m=d['ml_apply']; print('$ns', m['streams'], round(m['ms_per_batch'],4), round(m['roofline']['frac'],3))"; done
