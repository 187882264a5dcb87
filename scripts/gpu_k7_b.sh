#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
IVK_K7_SMEM=1 timeout 300 python scripts/time_k7.py cfg3 full,kron 3 > gpurun_out/k7_cfg3_smem.json 2> gpurun_out/k7_cfg3_smem.err
timeout 300 python scripts/time_k7.py cfg3 full,kron 5 > gpurun_out/k7_cfg3_reg.json 2> gpurun_out/k7_cfg3_reg.err
timeout 300 python scripts/time_k7.py cfg2 full,kron 5 > gpurun_out/k7_cfg2_reg.json 2> gpurun_out/k7_cfg2_reg.err
IVK_K7_SMEM=1 timeout 300 python scripts/time_k7.py cfg2 full,kron 3 > gpurun_out/k7_cfg2_smem.json 2> gpurun_out/k7_cfg2_smem.err
grep -h '"ms"' gpurun_out/k7_cfg3_smem.json | tail -4; grep -h '"ms"' gpurun_out/k7_cfg3_reg.json | tail -4
tail -3 gpurun_out/k7_cfg3_reg.err
