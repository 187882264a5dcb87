mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_full.log 2>&1; echo "exit $?" >> gpurun_out/pytest_full.log
