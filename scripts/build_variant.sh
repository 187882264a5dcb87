#!/bin/bash
# Build a libivk variant with extra nvcc flags into ab_libs/libivk_NAME.so
# (git-ignored, travels with gpurun).  usage: scripts/build_variant.sh NAME [-DMACRO=..]...
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
mkdir -p ab_libs
SRC=paper_2202_07381_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -o ab_libs/libivk_$NAME.so $SRC/ivk_operator.cu $SRC/ivk_patches.cu $SRC/ivk_transfer.cu \
  $SRC/ivk_coarse.cu $SRC/ivk_general.cu $SRC/ivk_krylov.cu $SRC/ivk_assembly.cu
echo built ab_libs/libivk_$NAME.so
