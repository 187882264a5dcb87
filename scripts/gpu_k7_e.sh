#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_CMD="python scripts/time_k7.py cfg3 full 3" AB_TAIL=40 AB_TAG=k7_e bash scripts/ab_run.sh cur k7_8x10 k7_32x3 k7_16m4 k7_16m2
grep -h '== \|"ms"' gpurun_out/ab_k7_e.log | tr '\n' ' '
