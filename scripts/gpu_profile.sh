mkdir -p gpurun_out
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-full-mode"
$CMD > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_bench.csv $CMD > gpurun_out/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"patch_apply_kron_kernel|stage_apply|patch_combine" -s 6 -c 3 -o gpurun_out/prof_bench $CMD > gpurun_out/ncu_full_bench.log 2>&1
echo done
