#!/bin/bash
# K3m fragment layout: parity on the modal paths + bench + ncu of K3m
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests/test_gpu_krylov.py tests/test_host_api.py tests/test_gpu_interop.py tests/test_gpu_coverage.py tests/test_gpu_parity.py tests/test_shard.py tests/test_modal.py -x -q -m gpu > gpurun_out/pytest_b.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_b.txt
IVK_PARITY_LOG=gpurun_out/parity_b.jsonl timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py -q -m gpu -k "cfg2 and modal" > gpurun_out/pytest_b_full.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_b_full.txt
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-full-mode > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err && \
ncu --set full --clock-control none --import-source on -k regex:patch_apply_modal_tc -s 20 -c 1 -o gpurun_out/prof_k3m_b python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-full-mode > gpurun_out/ncu_b.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_b.log
