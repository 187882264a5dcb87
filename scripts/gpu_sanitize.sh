#!/bin/bash
# compute-sanitizer over the small parity cases: memcheck, racecheck,
# synccheck, initcheck, restricted to libivk's kernels (namespace ivk).
# Logs -> gpurun_out/sanitize_<tool>.log.  usage: bash scripts/gpu_sanitize.sh [tools]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TOOLS=${1:-"memcheck racecheck synccheck initcheck"}
# crossed: every formulation (K1, K3 full/kron/kron-sym/dedup/modal, K4, K5, K6
# dense, K8, K9 via FGMRES, graph replay); coverage: K6 lu, modal any tableau;
# Krylov; assembly (K10); MHD 16^2 (K1g, K7g, K5g); 3-D (K7e/K3e wide, modal CTA);
# peer-memory K4p loopback.
SEL_PARITY='tests/test_gpu_parity.py -k crossed'
SEL_MISC='tests/test_gpu_coverage.py -k "coarse_methods and crossed or modal_any_tableau and radauiia-3"'
SEL_KRY='tests/test_gpu_krylov.py tests/test_gpu_assembly.py -k "crossed or relinearize or krylov or dot or mgs or fgmres or concurrent"'
SEL_MHD='tests/test_gpu_mhd.py -k "mhd16 and (operator_apply or sweep or transfers)"'
SEL_3D='tests/test_gpu_3d.py -k "matvec_and_sweep_3d and radauiia"'
SEL_PEER='tests/test_shard.py -k "peer_fused and s3-2-modal"'
for tool in $TOOLS; do
  LOG=gpurun_out/sanitize_$tool.log
  : > $LOG
  EXTRA=""
  [ $tool = initcheck ] && EXTRA="--track-unused-memory no"
  for sel in "$SEL_PARITY" "$SEL_MISC" "$SEL_KRY" "$SEL_MHD" "$SEL_3D" "$SEL_PEER"; do
    echo "### $tool: $sel" >> $LOG
    eval timeout 1500 compute-sanitizer --tool $tool $EXTRA --kernel-name regex:ivk \
      --error-exitcode 99 --print-limit 50 python -m pytest $sel -x -q -m gpu -p no:cacheprovider >> $LOG 2>&1
    echo "### rc=$?" >> $LOG
  done
done
