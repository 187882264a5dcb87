#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_k1tiles.py tests/test_gpu_parity.py -q -m gpu -x -k "k1tiles or operator_apply or sweep" > gpurun_out/pytest_k1t.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k1t.log
AB_TAG=k1t bash scripts/ab_run.sh cur:IVK_K1_TILES=0 cur:IVK_K1_TILES=128 cur:IVK_K1_TILES=256 cur:IVK_K1_TILES=512 \
  t256u8:IVK_K1_TILES=256 t256u8:IVK_K1_TILES=128 t512:IVK_K1_TILES=512 t512:IVK_K1_TILES=256 t160:IVK_K1_TILES=128 t320r80:IVK_K1_TILES=256
