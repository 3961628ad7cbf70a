#!/bin/bash
# A/B of the tridiagonalisation tail size (FKK_TRIDIAG_TAIL = cluster size, FKK_TRIDIAG_MT = tail columns)
mkdir -p gpurun_out
{
for c in 8 16; do
for mt in 150 250 340 440 600; do
  echo "== tail $c mt $mt"
  FKK_TRIDIAG_MT=$mt FKK_TRIDIAG_TAIL=$c timeout 120 python tools/eig_breakdown.py 1000 60 2>&1 | grep "tridiag"
done
done
} > gpurun_out/tri_mc.log 2>&1
cat gpurun_out/tri_mc.log
