#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py -q -m gpu -x -k "modal or sweep or vcycle" 2>&1 | tail -2
AB_TAG=k3m_swz bash scripts/ab_run.sh cur noswz
cat gpurun_out/ab_k3m_swz.log
