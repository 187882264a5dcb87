mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_krylov.py tests/test_gpu_assembly.py -x -q > gpurun_out/pytest_k.log 2>&1; echo "exit $?" >> gpurun_out/pytest_k.log
timeout 900 python bench.py --no-cpu-baseline --no-full-mode > gpurun_out/bench.log 2>&1; echo "exit $?" >> gpurun_out/bench.log
