mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest1.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke1.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke1.log
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench1.log 2>&1; echo "bench exit $?" >> gpurun_out/bench1.log
