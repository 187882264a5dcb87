#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_TAG=k3m_r96 bash scripts/ab_run.sh cur r96 r96:IVK_MODAL_CPS=5 r96ns r96:IVK_MODAL_CPS=3
cat gpurun_out/ab_k3m_r96.log
