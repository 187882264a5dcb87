#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_3d.py tests/test_setup3d.py -q -m gpu -x 2>&1 | tail -2
AB_CMD="python scripts/prof_general.py cfg4 12 modal" AB_TAG=cta_np AB_TIMEOUT=300 bash scripts/ab_run.sh ctapred cur
cat gpurun_out/ab_cta_np.log
