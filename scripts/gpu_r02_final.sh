#!/bin/bash
# Round-2 validation of HEAD: smoke, full GPU suite (incl. full-size parity and
# guard bands), default bench, reference arm, launch list of the bench command
# restricted to this library's kernels, --set full of the sweep kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r02final}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
nproc >> gpurun_out/smi_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
IVK_PARITY_LOG=gpurun_out/parity_$TAG.jsonl timeout 2400 python -m pytest tests/ -q -m gpu -s --durations=15 > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench exit $?" >> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref exit $?" >> gpurun_out/bench_ref_$TAG.err
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-full-mode"
timeout 600 $CMD > gpurun_out/bench_plain_$TAG.json 2> gpurun_out/bench_plain_$TAG.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:ivk:: -c 6000 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_launch_$TAG.log
for k in patch_apply_modal stage_apply_kernel patch_combine; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 60 -c 1 -o gpurun_out/prof_${TAG}_$k -f $CMD > gpurun_out/ncu_full_${TAG}_$k.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_${TAG}_$k.ncu-rep > gpurun_out/summary_${TAG}_$k.txt 2>&1
done
tail -3 gpurun_out/pytest_$TAG.log; cat gpurun_out/smoke_$TAG.log | tail -2; head -c 600 gpurun_out/bench_$TAG.json
