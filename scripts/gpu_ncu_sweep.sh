#!/bin/bash
# ncu --set full of the cfg2 fine-level sweep kernels (K1, K3m, K4) in
# scripts/prof_general.py, after a plain run of the same command; summaries
# + SASS hot lines to gpurun_out/.  usage: bash scripts/gpu_ncu_sweep.sh TAG [kernels]
cd $GRAFT_REPO_ROOT
TAG=${1:-sweep}
KS=${2:-"stage_apply_kernel patch_apply_modal_tc patch_combine_kernel"}
mkdir -p gpurun_out
CMD="python scripts/prof_general.py cfg2 6 modal"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || exit 1
for k in $KS; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_${TAG}_$k -f $CMD > gpurun_out/ncu_${TAG}_$k.log 2>&1
  echo "$k exit $?" >> gpurun_out/ncu_${TAG}.status
  python scripts/ncu_summary.py gpurun_out/prof_${TAG}_$k.ncu-rep > gpurun_out/summary_${TAG}_$k.txt 2>&1
  python scripts/sass_hot.py gpurun_out/prof_${TAG}_$k.ncu-rep 66049 > gpurun_out/sass_${TAG}_$k.txt 2>&1
done
