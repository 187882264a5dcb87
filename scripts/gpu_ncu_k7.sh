#!/bin/bash
# ncu --set full of the K7 kernels at the 66,049-patch level: usage gpu_ncu_k7.sh TAG CFG [env...]
cd $GRAFT_REPO_ROOT
TAG=$1; CFG=${2:-cfg3}; shift; shift
mkdir -p gpurun_out
for kv in "$@"; do export "$kv"; done
for mode in full kron; do
  CMD="python scripts/time_k7.py $CFG $mode 1"
  timeout 300 $CMD > gpurun_out/plain_k7_${TAG}_$mode.log 2>&1 || exit 1
  # one launch per level: skip the four smaller levels -> the 66,049-patch level
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:patch_factor -s 4 -c 1 \
    -o gpurun_out/prof_k7_${TAG}_$mode -f $CMD > gpurun_out/ncu_k7_${TAG}_$mode.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_k7_${TAG}_$mode.ncu-rep > gpurun_out/summary_k7_${TAG}_$mode.txt 2>&1
  python scripts/sass_hot.py gpurun_out/prof_k7_${TAG}_$mode.ncu-rep 66049 > gpurun_out/sass_k7_${TAG}_$mode.txt 2>&1
done
cat gpurun_out/summary_k7_${TAG}_*.txt
