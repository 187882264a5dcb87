#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_TAG=k1_order bash scripts/ab_run.sh cur:IVK_K1_ORDER=0 cur:IVK_K1_ORDER=1
cat gpurun_out/ab_k1_order.log
IVK_K1_ORDER=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
