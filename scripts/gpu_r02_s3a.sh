#!/bin/bash
# session 3 call A: MHD tests, sweep ncu (K1/K3m/K4), launch list of the bench
# command (libivk kernels only), cfg3 Newton phase breakdown.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mhd.py -q -m gpu -x > gpurun_out/pytest_mhd_s3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mhd_s3.log
timeout 900 bash scripts/gpu_ncu_sweep.sh s3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ivk --csv --log-file gpurun_out/launches_ivk_s3.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-full-mode > gpurun_out/ncu_launch_s3.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_launch_s3.log
timeout 900 python scripts/time_newton.py cfg3 2 > gpurun_out/newton_cfg3_s3.json 2> gpurun_out/newton_cfg3_s3.err; echo "rc=$?" >> gpurun_out/newton_cfg3_s3.err
