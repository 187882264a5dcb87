#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_TAG=share AB_TAIL=2 bash scripts/ab_run.sh cur cur:IVK_EXP_SHARE_RECORDS=1
cat gpurun_out/ab_share.log
