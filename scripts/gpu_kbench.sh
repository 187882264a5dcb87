mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "vcycle or graph" > gpurun_out/pytest_k.log 2>&1; echo "exit $?" >> gpurun_out/pytest_k.log
timeout 600 python scripts/kernel_bench.py 50 cfg2 > gpurun_out/kbench.log 2>&1; echo "exit $?" >> gpurun_out/kbench.log
ncu --set full --clock-control none --import-source on -k regex:"coarse_solve" -s 3 -c 1 -o gpurun_out/prof_coarse python scripts/kernel_bench.py 5 cfg2 > gpurun_out/ncu_coarse.log 2>&1
