#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py tests/test_gpu_mhd.py -q -m gpu -x > gpurun_out/pytest_k7.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_k7.log
tail -3 gpurun_out/pytest_k7.log
AB_CMD="python scripts/time_k7.py cfg3 full 3" AB_TAIL=40 AB_TAG=k7_d bash scripts/ab_run.sh cur k7_8x10 k7_32x3 k7_16m4
grep -h '== \|"ms"' gpurun_out/ab_k7_d.log | tr '\n' ' '
timeout 300 python scripts/time_k7.py cfg3 kron 5 > gpurun_out/k7_cfg3_reg3.json 2> gpurun_out/k7_cfg3_reg3.err
grep -h '"ms"' gpurun_out/k7_cfg3_reg3.json | tr '\n' ' '
