#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py tests/test_gpu_newton.py tests/test_gpu_mhd.py tests/test_gpu_assembly.py tests/test_gpu_mhd_relin.py -q -m gpu -x > gpurun_out/pytest_k7.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_k7.log
tail -5 gpurun_out/pytest_k7.log
IVK_K7_SMEM=1 timeout 300 python scripts/time_k7.py cfg3 full,kron 3 > gpurun_out/k7_cfg3_smem.json 2> gpurun_out/k7_cfg3_smem.err
timeout 300 python scripts/time_k7.py cfg3 full,kron 5 > gpurun_out/k7_cfg3_reg.json 2> gpurun_out/k7_cfg3_reg.err
timeout 300 python scripts/time_k7.py cfg2 full,kron 5 > gpurun_out/k7_cfg2_reg.json 2> gpurun_out/k7_cfg2_reg.err
IVK_K7_SMEM=1 timeout 300 python scripts/time_k7.py cfg2 full,kron 3 > gpurun_out/k7_cfg2_smem.json 2> gpurun_out/k7_cfg2_smem.err
grep -h '"ms"' gpurun_out/k7_cfg3_smem.json | tail -4; grep -h '"ms"' gpurun_out/k7_cfg3_reg.json | tail -4
