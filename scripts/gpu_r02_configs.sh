#!/bin/bash
# bench.py on the other BASELINE configs (HEAD), one JSON line each.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 1200 python bench.py --config $c --no-cpu-cycles > gpurun_out/bench_${c}_r02.json 2> gpurun_out/bench_${c}_r02.err; echo "$c exit $?" >> gpurun_out/bench_${c}_r02.err
  head -c 300 gpurun_out/bench_${c}_r02.json; echo
done
timeout 600 python scripts/time_newton.py cfg3 2 > gpurun_out/newton_cfg3_r02final.json 2> gpurun_out/newton_cfg3_r02final.err
grep -h '"seconds"' gpurun_out/newton_cfg3_r02final.json
