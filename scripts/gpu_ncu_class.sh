mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dedup or auto" > gpurun_out/pytest_k.log 2>&1; echo "exit $?" >> gpurun_out/pytest_k.log
CMD="python scripts/kernel_bench.py 50 cfg2 dedup"
$CMD > gpurun_out/kb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"patch_apply_class" -s 3 -c 1 -o gpurun_out/prof_class $CMD > gpurun_out/ncu_class.log 2>&1
echo "exit $?" >> gpurun_out/ncu_class.log
