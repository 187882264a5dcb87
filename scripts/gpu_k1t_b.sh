#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_k1tiles.py -q -m gpu -x > gpurun_out/pytest_k1t.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_k1t.log
[ $rc = 0 ] || exit 1
AB_TAG=k1t_c bash scripts/ab_run.sh cur:IVK_K1_TILES=0 cur:IVK_K1_TILES=48 cur:IVK_K1_TILES=64 cur:IVK_K1_TILES=96 cur:IVK_K1_TILES=128 cur:IVK_K1_TILES=192 cur:IVK_K1_TILES=256 \
  u8:IVK_K1_TILES=64 u8:IVK_K1_TILES=128 u2:IVK_K1_TILES=64 u2:IVK_K1_TILES=128
bash scripts/gpu_ncu_k1t.sh k1t_blob cur 128
