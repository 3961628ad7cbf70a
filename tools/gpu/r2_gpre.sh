mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "cfg4 or odd or gram or wide" > gpurun_out/gpre_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/gpre_tests.log
for c in 148 91; do echo "ctas=$c"; FKK_GRAM_CTAS=$c timeout 600 python tools/prof_cfg4.py 1000000 3 2>&1 | grep -v Warn | tail -1; done
timeout 300 python tools/prof_transform.py 703026 3 2>&1 | grep -v Warn | tail -1
