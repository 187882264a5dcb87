#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py tests/test_gpu_mhd.py tests/test_gpu_newton.py tests/test_gpu_assembly.py tests/test_gpu_mhd_relin.py tests/test_gpu_3d.py -q -m gpu -x > gpurun_out/pytest_k7.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_k7.log
tail -3 gpurun_out/pytest_k7.log
timeout 300 python scripts/time_k7.py cfg3 full,kron 5 > gpurun_out/k7_cfg3_reg5.json 2> gpurun_out/k7_cfg3_reg5.err
grep -h '"ms"' gpurun_out/k7_cfg3_reg5.json | tr '\n' ' '
timeout 300 python scripts/time_k7.py cfg2 full,kron 5 > gpurun_out/k7_cfg2_reg5.json 2> gpurun_out/k7_cfg2_reg5.err
grep -h '"ms"' gpurun_out/k7_cfg2_reg5.json | tr '\n' ' '
timeout 600 python scripts/time_newton.py cfg3 2 > gpurun_out/newton_cfg3_k7reg.json 2> gpurun_out/newton_cfg3_k7reg.err
grep -h 'seconds\|relinearize\|K10\|fgmres"' gpurun_out/newton_cfg3_k7reg.json | tr '\n' ' '
bash scripts/gpu_ncu_k7.sh reg5 cfg3 > /dev/null
bash scripts/gpu_ncu_k7.sh reg5c2 cfg2 > /dev/null
cat gpurun_out/summary_k7_reg5*_full.txt | grep "Kernel Name\|duration\|fp64"
