# ncu of the general-path / wide-block sweep kernels (cfg5 MHD, cfg4 3-D):
# plain run first (must exit 0), then one --set full capture per kernel.
mkdir -p gpurun_out
for c in cfg5 cfg4; do
  CMD="python scripts/prof_general.py $c 6"
  $CMD > gpurun_out/prof_${c}_plain.log 2>&1 || { echo "$c plain run failed"; continue; }
  for k in general_apply_kernel stage_apply patch_apply_kron_wide patch_combine; do
    ncu --set full --clock-control none --import-source on -k regex:"$k" -s 2 -c 1 \
      -o gpurun_out/prof_${c}_$k $CMD > gpurun_out/ncu_${c}_$k.log 2>&1
    echo "$c $k exit $?" >> gpurun_out/ncu_general.log
  done
done
