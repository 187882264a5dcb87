#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_3d.py -q -m gpu -x 2>&1 | tail -2
AB_TAG=k3m_ch bash scripts/ab_run.sh cur k3mch2
cat gpurun_out/ab_k3m_ch.log
AB_CMD="python scripts/prof_general.py cfg4 12 modal" AB_TAG=cta_ch3 AB_TIMEOUT=300 bash scripts/ab_run.sh cur
cat gpurun_out/ab_cta_ch3.log
