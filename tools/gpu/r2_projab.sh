# A/B of the projection's TMEM split: 2 accumulator sets x 2 A slots (default) vs 1 set x 2/3/4 A slots
for v in "" 2 3 4; do
  if [ -z "$v" ]; then echo "default"; timeout 300 python tools/prof_transform.py 703026 3 2>&1 | grep -v Warn | tail -1;
  else echo "NBUF=1 NA=$v"; FKK_PROJECT_NBUF=$v timeout 300 python tools/prof_transform.py 703026 3 2>&1 | grep -v Warn | tail -1; fi
done
