#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python scripts/prof_general.py cfg4 6 modal"
timeout 300 $CMD > gpurun_out/plain_cta.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:patch_apply_modal_cta -s 3 -c 1 -o gpurun_out/prof_cta -f $CMD > gpurun_out/ncu_cta.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_cta.ncu-rep > gpurun_out/summary_cta.txt 2>&1
python scripts/ncu_lines.py gpurun_out/prof_cta.ncu-rep 35937 40 > gpurun_out/lines_cta.txt 2>&1
cat gpurun_out/summary_cta.txt; head -45 gpurun_out/lines_cta.txt
