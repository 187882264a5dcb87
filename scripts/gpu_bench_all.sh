mkdir -p gpurun_out
for c in cfg1 cfg3; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "exit $?" >> gpurun_out/bench_$c.log
done
timeout 600 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_ref.log 2>&1; echo "exit $?" >> gpurun_out/bench_ref.log
