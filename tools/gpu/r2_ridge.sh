# cfg4 geometry: stage split (Gram split rule with a full last wave; fPEC ridge at k = 100 in shared memory)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "cfg4 or wide or odd_channel or image_gram" > gpurun_out/ridge_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/ridge_tests.log
for i in 1 2; do timeout 300 python tools/prof_cfg4.py 1000000 3 2>&1 | grep -v Warn | tail -1 | cut -c1-300; done
