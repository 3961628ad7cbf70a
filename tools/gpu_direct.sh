# direct-path parity tests + per-kernel times at cfg3 rows (131,072-spectrum batch)
mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "direct" 2>&1 | tail -2
timeout 300 python tools/kernel_breakdown.py --what direct --rows 131072 --reps 2 2>&1 | grep -v Warn | head -8
} > gpurun_out/direct.log 2>&1
cat gpurun_out/direct.log
