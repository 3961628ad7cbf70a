#!/bin/bash
# parity tests of the fKK path + stage times (cfg3) + optional env A/B: gpu_quick.sh "ENV=val ..."
mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -v "^\s*$" | grep "Error\|error\|assert\|passed\|failed" | head -20
timeout 300 python tools/time_eig.py cfg3 2>&1 | tail -1
for e in "$@"; do echo "== $e"; env $e timeout 300 python tools/time_eig.py cfg3 2>&1 | tail -1; done
} > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log
