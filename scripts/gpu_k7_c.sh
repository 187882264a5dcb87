#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py tests/test_gpu_mhd.py tests/test_gpu_3d.py -q -m gpu -x > gpurun_out/pytest_k7.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_k7.log
tail -5 gpurun_out/pytest_k7.log
timeout 300 python scripts/time_k7.py cfg3 full,kron 5 > gpurun_out/k7_cfg3_reg2.json 2> gpurun_out/k7_cfg3_reg2.err
timeout 300 python scripts/time_k7.py cfg2 full,kron 5 > gpurun_out/k7_cfg2_reg2.json 2> gpurun_out/k7_cfg2_reg2.err
grep -h '"ms"' gpurun_out/k7_cfg3_reg2.json | tr '\n' ' '
grep -h '"ms"' gpurun_out/k7_cfg2_reg2.json | tr '\n' ' '
bash scripts/gpu_ncu_k7.sh reg2 cfg3
