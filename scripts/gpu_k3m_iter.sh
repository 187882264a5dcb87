#!/bin/bash
# K3m iteration: modal parity (small + cfg2 full-vector), bench (no CPU leg),
# then ncu of one K3m launch.  usage: bash scripts/gpu_k3m_iter.sh TAG
TAG=${1:-iter}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py tests/test_shard.py -x -q -m gpu -k "modal or auto or Loopback or loopback or tableau" > gpurun_out/pytest_$TAG.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_$TAG.txt
IVK_PARITY_LOG=gpurun_out/parity_$TAG.jsonl timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py -q -m gpu -k "cfg2 and modal" >> gpurun_out/pytest_$TAG.txt 2>&1
echo "full rc=$?" >> gpurun_out/pytest_$TAG.txt
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-full-mode > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err && \
ncu --set full --clock-control none --import-source on -k regex:patch_apply_modal_tc -s 20 -c 1 -o gpurun_out/prof_k3m_$TAG python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-full-mode > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
