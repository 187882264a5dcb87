#!/bin/bash
# A/B of the K3m (modal, tensor-core) kernel on cfg2: the libraries under
# ab_libs/ (old / new builds) and CTA shapes given as KB:CPS pairs
# (IVK_MODAL_CTA_KB smem budget per CTA, IVK_MODAL_CPS CTAs per SM).
set -u
LIB=paper_2202_07381_b200/libivk.so
cp $LIB /tmp/libivk_cur.so
for v in ${VARIANTS:-old new}; do
  [ -f ab_libs/libivk_$v.so ] || continue
  cp ab_libs/libivk_$v.so $LIB
  for shape in ${SHAPES:-72:3 59:3 94:2 48:4}; do
    kb=${shape%%:*}; cps=${shape##*:}
    echo "== $v KB=$kb CPS=$cps"
    IVK_MODAL_CTA_KB=$kb IVK_MODAL_CPS=$cps timeout 300 python scripts/prof_general.py cfg2 12 modal 2>&1 | tail -1
  done
done
cp /tmp/libivk_cur.so $LIB
