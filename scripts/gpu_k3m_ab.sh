#!/bin/bash
# K3m iteration with CTA-shape A/B: parity, bench under env variants, ncu default.
TAG=${1:-ab}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py tests/test_shard.py -x -q -m gpu -k "modal or auto or Loopback or loopback or tableau" > gpurun_out/pytest_$TAG.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_$TAG.txt
IVK_PARITY_LOG=gpurun_out/parity_$TAG.jsonl timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py -q -m gpu -k "cfg2 and modal" >> gpurun_out/pytest_$TAG.txt 2>&1
echo "full rc=$?" >> gpurun_out/pytest_$TAG.txt
for v in "" "IVK_MODAL_CPS=5 IVK_MODAL_CTA_KB=41" "IVK_MODAL_CPS=4 IVK_MODAL_CTA_KB=41" "IVK_MODAL_CPS=3 IVK_MODAL_CTA_KB=72" "IVK_MODAL_CPS=2 IVK_MODAL_CTA_KB=100"; do
  echo "== $v" >> gpurun_out/ab_$TAG.txt
  env $v python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-full-mode 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['value'],d['roofline']['avg_launch_ms'],d['vcycle_ms'])" >> gpurun_out/ab_$TAG.txt
done
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-full-mode > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err && \
ncu --set full --clock-control none --import-source on -k regex:patch_apply_modal_tc -s 20 -c 1 -o gpurun_out/prof_k3m_$TAG python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-full-mode > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
