#!/bin/bash
# Generic A/B on the GPU box: for each "LIBNAME[:ENV=VAL,...]" argument run
# CMD (env AB_CMD, default: prof_general cfg2 40 modal) with that library
# variant (ab_libs/libivk_LIBNAME.so; "cur" = the in-tree build) and env.
# Output: gpurun_out/ab_${AB_TAG}.log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
LIB=paper_2202_07381_b200/libivk.so
CMD=${AB_CMD:-"python scripts/prof_general.py cfg2 40 modal"}
TAG=${AB_TAG:-run}
cp $LIB /tmp/libivk_cur.so
for rep in 1 2; do
for spec in "$@"; do
  name=${spec%%:*}
  envs=""
  [[ "$spec" == *:* ]] && envs=$(echo "${spec#*:}" | tr ',' ' ')
  if [ "$name" = cur ]; then cp /tmp/libivk_cur.so $LIB; else cp ab_libs/libivk_$name.so $LIB; fi
  echo "== $spec rep $rep"
  env $envs timeout ${AB_TIMEOUT:-150} $CMD 2>&1 | tail -${AB_TAIL:-1}
done
done > gpurun_out/ab_$TAG.log 2>&1
cp /tmp/libivk_cur.so $LIB
