#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py tests/test_gpu_guards.py -q -m gpu -x -k "modal or sweep or vcycle or guards or bounds" 2>&1 | tail -2
AB_TAG=k3m_micro bash scripts/ab_run.sh prev cur
cat gpurun_out/ab_k3m_micro.log
