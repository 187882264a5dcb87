# HEAD validation (scripts/gpu_validate.sh) followed by the bench launch list
# and --set full captures of K3m / K1 / K4 (scripts/gpu_ncu_bench.sh).
bash scripts/gpu_validate.sh
bash scripts/gpu_ncu_bench.sh > gpurun_out/ncu_bench.log 2>&1
