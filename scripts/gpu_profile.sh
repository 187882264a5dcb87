mkdir -p gpurun_out
python scripts/prof_workload.py cfg2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python scripts/prof_workload.py cfg2 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"patch_apply|stage_apply|patch_combine|transfer|coarse_solve" -s 0 -c 8 -o gpurun_out/prof_cfg2 python scripts/prof_workload.py cfg2 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:"patch_factor" -s 5 -c 1 -o gpurun_out/prof_factor python scripts/prof_workload.py cfg2 > gpurun_out/ncu_factor.log 2>&1
echo done
