mkdir -p gpurun_out
CMD="python scripts/kernel_bench.py 5 cfg2 kron"
$CMD > gpurun_out/kb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stage_apply_kernel|patch_combine" -s 2 -c 2 -o gpurun_out/prof_k1 $CMD > gpurun_out/ncu_k1.log 2>&1
echo "exit $?" >> gpurun_out/ncu_k1.log
