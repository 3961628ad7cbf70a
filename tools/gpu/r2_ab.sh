# factorized path A/B (phase bit masks instead of indexed arrays: no local memory in the Gram /
# projection / reconstruction pipelines; reconstruction output boxes triple-buffered)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "not direct and not als and not conventional" > gpurun_out/ab_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/ab_tests.log
for v in new head new head; do
  if [ $v = head ]; then export FKK_LIB=$PWD/paper_2005_07132_b200/lib/libfkk_head.so; else unset FKK_LIB; fi
  timeout 600 python tools/time_eig.py 703026 10 2>&1 | grep -v Warn | tail -1 | sed "s/^/$v /"
done
