#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_TAG=k1cs bash scripts/ab_run.sh cur k1cs
cat gpurun_out/ab_k1cs.log
