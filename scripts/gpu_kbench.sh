mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coverage.py -q > gpurun_out/pytest_k.log 2>&1; echo "exit $?" >> gpurun_out/pytest_k.log
