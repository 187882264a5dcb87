mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dedup or auto" > gpurun_out/pytest_k.log 2>&1; echo "exit $?" >> gpurun_out/pytest_k.log
timeout 600 python scripts/kernel_bench.py 50 cfg2 kron,dedup > gpurun_out/kbench.log 2>&1; echo "exit $?" >> gpurun_out/kbench.log
