for e in FKK_PROJECT_NBUF=2 FKK_PROJECT_NBUF=2 FKK_PROJECT_NBUF=4 FKK_PROJECT_NBUF=4 X=1 X=2; do
  echo "== $e"; env $e timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "factorized_cfg2" 2>&1 | grep "AssertionError\|passed\|failed" | head -3
done
