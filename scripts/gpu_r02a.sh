#!/bin/bash
# round-2 validation: changed GPU tests, full-size parity, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests/test_gpu_krylov.py tests/test_host_api.py tests/test_gpu_interop.py tests/test_gpu_coverage.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_changed.txt 2>&1
echo "changed rc=$?" >> gpurun_out/pytest_changed.txt
IVK_PARITY_LOG=gpurun_out/parity_fullsize.jsonl timeout 1500 python -m pytest tests/test_gpu_fullsize_parity.py -q -m gpu -s --durations=0 > gpurun_out/pytest_fullsize_parity.txt 2>&1
echo "fullsize rc=$?" >> gpurun_out/pytest_fullsize_parity.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
echo "bench rc=$?" >> gpurun_out/bench_r02a.err
