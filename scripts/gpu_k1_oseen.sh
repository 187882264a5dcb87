#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_CMD="python scripts/prof_general.py cfg3 10 kron" AB_TAG=k1_oseen2 AB_TIMEOUT=400 bash scripts/ab_run.sh cur uj5 uj6
cat gpurun_out/ab_k1_oseen2.log
