mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_assembly.py -x -q > gpurun_out/pytest_k.log 2>&1; echo "exit $?" >> gpurun_out/pytest_k.log
