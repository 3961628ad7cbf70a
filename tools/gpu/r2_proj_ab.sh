# projection TMEM split: 2 accumulator sets + 2 A slots (default) vs 1 set + 3..5 A slots
mkdir -p gpurun_out
for v in default 3 5 default; do
  if [ $v = default ]; then unset FKK_PROJECT_NBUF; else export FKK_PROJECT_NBUF=$v; fi
  timeout 600 python tools/time_eig.py 703026 10 2>&1 | grep -v Warn | tail -1 | sed "s/^/nbuf=$v /" | cut -c1-200
done
