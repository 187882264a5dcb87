# ncu --set full of the fine-level K1 (cfg2) after a plain run of the same command.
mkdir -p gpurun_out
CMD="python scripts/prof_general.py cfg2 6 modal"
$CMD > gpurun_out/k1_fine_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:stage_apply_kernel -s 3 -c 1 -o gpurun_out/prof_k1_fine -f $CMD > gpurun_out/ncu_k1_fine.log 2>&1
echo "k1 exit $?"
