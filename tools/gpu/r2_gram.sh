# balanced CTA-pair Gram: Gram-path parity tests, then the transform stage split at cfg3
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "gram or cfg3 or cfg4 or factorized or conventional or range or eq9 or floor or paper or smoke or host or ml" > gpurun_out/gram_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gram_tests.log
timeout 300 python tools/prof_transform.py 703026 5 2>&1 | grep -v Warn | tail -1
FKK_GRAM_DBG=1 timeout 300 python tools/prof_transform.py 703026 1 2>&1 | grep "gram_pre2 dbg" | tail -1
