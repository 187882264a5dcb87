#!/bin/bash
# ncu --set full of the tiled K1 kernel: usage gpu_ncu_k1t.sh TAG LIBNAME TILEROWS
cd $GRAFT_REPO_ROOT
TAG=$1; LIBN=$2; TR=$3
mkdir -p gpurun_out
LIB=paper_2202_07381_b200/libivk.so
cp $LIB /tmp/libivk_cur.so
[ "$LIBN" = cur ] || cp ab_libs/libivk_$LIBN.so $LIB
export IVK_K1_TILES=$TR
CMD="python scripts/prof_general.py cfg2 6 modal"
timeout 200 $CMD > gpurun_out/plain_$TAG.log 2>&1 || { cp /tmp/libivk_cur.so $LIB; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_apply -s 3 -c 1 -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_$TAG.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep > gpurun_out/summary_$TAG.txt 2>&1
python scripts/sass_hot.py gpurun_out/prof_$TAG.ncu-rep 1 > gpurun_out/sass_$TAG.txt 2>&1
cp /tmp/libivk_cur.so $LIB
