mkdir -p gpurun_out
CMD="python scripts/kernel_bench.py 5 cfg2 dedup"
$CMD > gpurun_out/kb_plain.log 2>&1 || exit 1
for k in stage_apply_kernel patch_apply_class patch_combine dense_gemv; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 -o gpurun_out/prof_r01_$k $CMD > gpurun_out/ncu_r01_$k.log 2>&1
  echo "$k exit $?" >> gpurun_out/ncu_r01.log
done
