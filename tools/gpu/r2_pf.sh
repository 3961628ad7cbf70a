# direct-path kernel variants: parity subset + cfg3 timing against the HEAD library (alternating)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "direct or conventional or wide or paper or clamp" > gpurun_out/pf_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/pf_tests.log
for v in new head new head; do
  if [ $v = head ]; then export FKK_LIB=$PWD/paper_2005_07132_b200/lib/libfkk_head.so; else unset FKK_LIB; fi
  timeout 600 python tools/prof_direct.py 703026 3 2>&1 | grep -v Warn | tail -1 | sed "s/^/$v /"
done
