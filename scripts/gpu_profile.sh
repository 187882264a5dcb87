mkdir -p gpurun_out
python scripts/prof_workload.py cfg2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python scripts/prof_workload.py cfg2 > gpurun_out/ncu_launch.log 2>&1
echo done
