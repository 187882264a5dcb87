mkdir -p gpurun_out
timeout 600 python scripts/kernel_bench.py 50 cfg2 > gpurun_out/kbench.log 2>&1; echo "exit $?" >> gpurun_out/kbench.log
ncu --set full --clock-control none --import-source on -k regex:"kron_sym" -s 3 -c 1 -o gpurun_out/prof_sym python scripts/kernel_bench.py 5 cfg2 > gpurun_out/ncu_sym.log 2>&1
