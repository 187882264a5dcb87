#!/bin/bash
# Round-2 validation of HEAD: full GPU suite (incl. full-size parity), smoke,
# default bench, reference arm, launch list of the bench command.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
nproc >> gpurun_out/smi_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
IVK_PARITY_LOG=gpurun_out/parity_$TAG.jsonl timeout 2400 python -m pytest tests/ -q -m gpu -s --durations=15 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench exit $?" >> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref exit $?" >> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-full-mode > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_launch_$TAG.log
