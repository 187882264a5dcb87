#!/bin/bash
# A/B of K1 on cfg2: cur (pipelined velocity rows, batches of 4) vs u3 (batches of 3, IVK_K1_U=3)
# from ab_libs/
mkdir -p gpurun_out
LIB=paper_2202_07381_b200/libivk.so
cp $LIB /tmp/libivk_cur.so
for rep in 1 2; do
for v in cur u3; do
  cp ab_libs/libivk_$v.so $LIB
  echo "== $v rep $rep"
  timeout 300 python scripts/prof_general.py cfg2 40 modal 2>&1 | tail -1
done
done > gpurun_out/ab_k1_u3.log 2>&1
cp /tmp/libivk_cur.so $LIB
