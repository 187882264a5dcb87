# ncu --set full of K3m (modal) on cfg2, after a plain run of the same command
python scripts/prof_general.py cfg2 4 modal > gpurun_out/pm_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:patch_apply_modal_tc -s 2 -c 1 \
  -o gpurun_out/prof_modal_cfg2 -f python scripts/prof_general.py cfg2 4 modal > gpurun_out/ncu_modal.log 2>&1
tail -1 gpurun_out/ncu_modal.log
