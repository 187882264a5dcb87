# Launch list of the headline bench command and one --set full capture of its
# top kernel (K3m), each after the same command exited 0 without ncu.
mkdir -p gpurun_out
CMD="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-full-mode"
$CMD > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_cfg2_modal.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?"
ncu --set full --clock-control none --import-source on -k regex:patch_apply_modal -s 60 -c 1 -o gpurun_out/prof_bench_k3m -f $CMD > gpurun_out/ncu_full_bench.log 2>&1
echo "full exit $?"
ncu --set full --clock-control none --import-source on -k regex:stage_apply_kernel -s 60 -c 1 -o gpurun_out/prof_bench_k1 -f $CMD > gpurun_out/ncu_full_bench_k1.log 2>&1
echo "k1 exit $?"
ncu --set full --clock-control none --import-source on -k regex:patch_combine -s 60 -c 1 -o gpurun_out/prof_bench_k4 -f $CMD > gpurun_out/ncu_full_bench_k4.log 2>&1
echo "k4 exit $?"
