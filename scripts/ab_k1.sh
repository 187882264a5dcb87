#!/bin/bash
# A/B of the fine-level K1 (stage_apply) on cfg2 over the libraries in
# ab_libs/ (old = current build, new = IVK_K1_PIPE, new4 = IVK_K1_PIPE with a
# 64-register cap), then the bench's e2e leg with 2 / 3 / 4 stream slots.
mkdir -p gpurun_out
LIB=paper_2202_07381_b200/libivk.so
cp $LIB /tmp/libivk_cur.so
for rep in 1 2; do
for v in old new new4; do
  cp ab_libs/libivk_$v.so $LIB
  echo "== $v rep $rep"
  timeout 300 python scripts/prof_general.py cfg2 40 modal 2>&1 | tail -1
done
done > gpurun_out/ab_k1.log 2>&1
cp /tmp/libivk_cur.so $LIB
for n in 2 3 4; do
  IVK_BENCH_E2E_SLOTS=$n timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-full-mode > gpurun_out/bench_slots$n.json 2> gpurun_out/bench_slots$n.err
done
