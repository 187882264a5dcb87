# DRAM traffic of the headline K3 kernels of cfg4 (modal, CTA kernel) and
# cfg5 (kron, wide kernel) for profiles/traffic.json; plain runs first.
mkdir -p gpurun_out
python scripts/prof_general.py cfg4 3 modal > gpurun_out/t4.log 2>&1 && \
ncu --set full --clock-control none -k regex:patch_apply_modal_cta -s 1 -c 1 -o gpurun_out/prof_traffic_cfg4 -f \
  python scripts/prof_general.py cfg4 3 modal > gpurun_out/ncu_t4.log 2>&1
echo "cfg4 $?"
python scripts/prof_general.py cfg5 3 kron > gpurun_out/t5.log 2>&1 && \
ncu --set full --clock-control none -k regex:patch_apply_kron_wide -s 1 -c 1 -o gpurun_out/prof_traffic_cfg5 -f \
  python scripts/prof_general.py cfg5 3 kron > gpurun_out/ncu_t5.log 2>&1
echo "cfg5 $?"
