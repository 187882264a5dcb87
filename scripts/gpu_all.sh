mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest.log
timeout 600 python scripts/kernel_bench.py 50 cfg2 kron,dedup > gpurun_out/kbench.log 2>&1; echo "exit $?" >> gpurun_out/kbench.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
